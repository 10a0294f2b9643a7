import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def golden_names():
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith(("nbr_", "growth_")))   # query / behaviour fixtures


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def pool_from_golden(g):
    from paper_2105_00039_b200.pool import AgentPool
    return AgentPool(position_x=g["in_px"].copy(), position_y=g["in_py"].copy(),
                     position_z=g["in_pz"].copy(), diameter=g["in_diam"].copy(),
                     adherence=g["in_adh"].copy(), uid=g["in_uid"].copy())


def params_from_golden(g):
    from paper_2105_00039_b200.mechanics import ForceParams
    k, ga, dt, md, ad = (float(v) for v in g["params"])
    return ForceParams(kappa=k, gamma=ga, timestep=dt, max_displacement=md, adherence_scale=ad)


def ir_from_golden(g):
    ir = float(g["interaction_radius"])
    return None if np.isnan(ir) else ir


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def cuda_required():
    if not has_cuda():
        pytest.skip("no CUDA device")
