"""Parity of the opt-in tensor-core ARM kernel (arm_tc.cu: tcgen05 kind::tf32,
3xTF32 split) against the fp64 oracle.  The path is chosen once
per process from CCRD_ARM_PATH, so the checks run in a subprocess
(tests/helpers/arm_tc_parity.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.timeout(600)
@pytest.mark.parametrize("variant", ["warpgroup", "warpgroup_ldg", "warp_specialised", "serial"])
def test_arm_tensor_core_path_matches_oracle(variant):
    """warpgroup: arm_tcg_kernel, the default tensor-core ARM (TMA window loads
    where every grid's rows are 16-byte strided, LDG staging elsewhere);
    warpgroup_ldg: the same with TMA off (CCRD_ARM_NO_TMA=1);
    warp_specialised: arm_tcw_kernel (CCRD_ARM_TC_WS=1); serial: arm_tc_kernel
    (CCRD_ARM_TC_SS=1)."""
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, CCRD_ARM_PATH="tc", CCRD_ARM_TC_SS="1" if variant == "serial" else "0",
               CCRD_ARM_TC_WS="1" if variant == "warp_specialised" else "0",
               CCRD_ARM_NO_TMA="1" if variant == "warpgroup_ldg" else "0")
    r = subprocess.run([sys.executable, os.path.join(here, "helpers", "arm_tc_parity.py")], env=env,
                       capture_output=True, text=True, timeout=540)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "arm_tc parity ok" in r.stdout
