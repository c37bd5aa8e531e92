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
@pytest.mark.parametrize("variant", ["pingpong", "pingpong_ldg", "warpgroup", "warpgroup_ldg"])
def test_arm_tensor_core_path_matches_oracle(variant):
    """pingpong: arm_tcp_kernel, the default tensor-core ARM (two blocks in
    flight per warpgroup; TMA window loads where every grid's rows are
    16-byte strided, LDG staging elsewhere); warpgroup: arm_tcg_kernel (one
    block per warpgroup, CCRD_ARM_TC_PP=0); *_ldg: TMA off (CCRD_ARM_NO_TMA=1)."""
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, CCRD_ARM_PATH="tc", CCRD_ARM_NO_TMA="1" if variant.endswith("_ldg") else "0",
               CCRD_ARM_TC_PP="0" if variant.startswith("warpgroup") else "1")
    r = subprocess.run([sys.executable, os.path.join(here, "helpers", "arm_tc_parity.py")], env=env,
                       capture_output=True, text=True, timeout=540)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "arm_tc parity ok" in r.stdout
