"""CPU oracle for the mechanical-interaction step -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package; the product path
(paper_2105_00039_b200) never does.  See oracle/cg_oracle.c for the restated
reference functions and DESIGN.md ("Oracle") for how it is pinned.
"""

from . import behavior
from .oracle import (OracleError, OracleGridOverflow, OracleStep, all_pairs, box_ids,
                     build, csr, force_phase, geometry, lib, morton_encode, morton_perm, neighbor_csr, step)

__all__ = ["behavior", "OracleError", "OracleGridOverflow", "OracleStep", "all_pairs", "box_ids", "build",
           "csr", "force_phase", "geometry", "lib", "morton_encode", "morton_perm", "step"]
