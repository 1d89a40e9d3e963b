"""GPU: the C++ shim of INTEGRATION.md, compiled verbatim against the reference's
own headers (oracle/_ref/integration_check, built by `make -C oracle
integration` where the reference sources exist), runs sweep1d::LaunchConfig
through the B200 library and must equal sweep1d::run_serial bit for bit."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "integration_check")


@pytest.mark.skipif(not os.path.exists(EXE), reason="integration_check not built (needs the reference sources)")
def test_integration_shim_is_a_bitwise_drop_in(gpu):
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and r.stdout.count("ok ") == 6
