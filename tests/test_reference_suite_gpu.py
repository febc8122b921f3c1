"""Drop-in proof: the reference's OWN unit tests (proj/tests/test_*.cpp, 62
cases / 6032 checks) linked against the reference objects whose hot-path
entry points (build_tree, associate_adaptive, make_virtual_points,
solve_mstep, register_with_tree, register_clouds) are replaced by the B200
adapter (paper_1807_02587_b200/adapter) -- built by `make -C oracle
ref-tests-b200` where /root/reference exists, run here on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests_b200")


def test_reference_unit_tests_through_b200_adapter():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/ref_unit_tests_b200 not built")
    env = dict(os.environ, TRG_ADAPTER_REPORT="1")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "| 0 failed |" in r.stdout
    line = [l for l in r.stderr.splitlines() if l.startswith("trg adapter:")]
    assert line and int(line[0].split()[2]) > 100, r.stderr[-2000:]
