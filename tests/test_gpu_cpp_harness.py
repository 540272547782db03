"""C++ lockstep parity: the unmodified reference core and the B200 engine in
one process (tests/cpp/parity_harness.cpp), through the reference's own C++
API on one side and the C++ facade include/bpsched_cuda.hpp on the other.

The binary is built where /root/reference exists (`make -C oracle harness`,
part of __graft_entry__.build()) and travels to the GPU box in oracle/_ref/."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HARNESS = os.path.join(ROOT, "oracle", "_ref", "parity_harness")


def test_cpp_lockstep_harness():
    if not os.path.exists(HARNESS):
        pytest.skip("oracle/_ref/parity_harness not built (needs /root/reference at build time)")
    p = subprocess.run([HARNESS], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    failed = [l for l in p.stdout.splitlines() if l.startswith("[FAIL]")]
    assert p.returncode == 0 and not failed, "\n".join(failed) or p.stderr
    assert "summary:" in p.stdout
