"""The reference's strategy types on the drop-in API (no GPU needed): labels
and validation as in reference engine.py:57-97, and every one of them maps to
the B200 path (as_gpu) in uid summation -- bit-identical to the reference's
strategies (run on the device in tests/test_gpu_parity.py)."""

import pytest

import paper_2105_00039_b200 as P


def test_labels_match_the_reference():
    assert P.strategy_label(P.Serial()) == "serial"
    assert P.strategy_label(P.AgentParallel(8)) == "parallel(8)"
    assert P.strategy_label(P.VoxelTiled(4)) == "voxel(4)"
    assert P.strategy_label(P.Gpu(1)) == "gpu(1)"
    with pytest.raises(TypeError):
        P.strategy_label(object())


def test_validation_matches_the_reference():
    with pytest.raises(ValueError):
        P.AgentParallel(0)
    with pytest.raises(ValueError):
        P.VoxelTiled(0)
    with pytest.raises(ValueError):
        P.VoxelTiled(2, tile_stencil_capacity=0)


def test_cpu_strategies_execute_on_the_b200_in_uid_order():
    for s in (P.Serial(), P.AgentParallel(16), P.VoxelTiled(2)):
        g = P.as_gpu(s)
        assert isinstance(g, P.Gpu) and g.device == 0 and g.summation == "uid"
        P.SimulationConfig(strategy=s)   # accepted
    assert P.as_gpu(P.Gpu(0, "stencil")).summation == "stencil"
    # an explicit tile capacity is a VoxelTiled-only contract (TileCapacityError): rejected up front
    with pytest.raises(NotImplementedError):
        P.SimulationConfig(strategy=P.VoxelTiled(2, tile_stencil_capacity=64))
    with pytest.raises(TypeError):
        P.SimulationConfig(strategy="serial")
