"""The reference's own C++ API on both sides of the boundary: the unmodified
parorb::opt_par_mod_inner vs parorb::gpu::opt_par_mod_inner (integration/
parorb_gpu_adapter.hpp over include/parorb_gpu.h), same Problem, same start."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
DEMO = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                    "dropin_demo")


@pytest.mark.skipif(not os.path.exists(DEMO), reason="dropin_demo is built only where /root/reference exists")
@pytest.mark.parametrize("args", [("16", "4", "12"), ("24", "6", "10"), ("9", "4", "6", "2")])
def test_reference_api_dropin(args):
    r = subprocess.run([DEMO, *args], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "OK" in r.stdout.strip().split("\n")[-1]
