"""XL class fallbacks, bit-exact against the oracle.

With the default 224 KB of dynamic shared memory C4's working sets fit, so the
XL kernel's fallback paths -- quantum steps on the HBM arena (`xl_step`),
warp-0 window begin / epoch / place_batch when the CTA scratch is too small --
would go untested.  `gs_set_xl_smem` shrinks the CTA's working-set budget to
force them.
"""
import pytest

from parity import assert_gpu_matches_oracle
from paper_2309_00558_b200 import backend, workloads as wl
from paper_2309_00558_b200.scenario import Scenario

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kb", [16, 40, 96])
def test_gpu_xl_fallbacks_match_oracle(kb):
    scen = [Scenario.from_dict(wl.c4(s, windows=25)) for s in range(2)]
    scen += [Scenario.from_dict(wl.c4(5, windows=12, n_funcs=80, fleet=40))]
    try:
        assert backend.set_xl_smem(kb * 1024) == kb * 1024
        assert_gpu_matches_oracle(scen, ["fast", "timeshare", "fast"])
    finally:
        backend.set_xl_smem(0)
