"""The reference's own C++ test cases compiled against the mirrored mswave::
API (include/mswave/*.hpp) and linked to libmswave_b200.so."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "test_mirror")


def test_cpp_mirror_builds():
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_cpp_mirror_reference_cases():
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failed" in out.stdout
