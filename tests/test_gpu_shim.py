"""Link-time drop-in: oracle/_ref/libbpsched_cuda_shim.so
defines bpsched::run (schedulers.hpp:156) over the B200 engine.  Preloaded into
a process that uses the UNMODIFIED reference core (oracle/_ref, built from
/root/reference), the reference's own callers of bpsched::run -- here its C
wrapper ref_run -- run on the device without a source change."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "oracle", "_ref", "libbpsched_cuda_shim.so")

PROG = r"""
import ctypes, json, sys
sys.path.insert(0, %r)
from oracle import pyoracle as po
# a C++ caller links the reference at link time; ctypes loads it RTLD_LOCAL
# unless asked, which would hide the reference's symbols from the shim
ctypes.CDLL(po.PATHS["ref"], mode=ctypes.RTLD_GLOBAL)
ref = po.load("ref")
out = {}
for kind, n, c, seed in (("lbp", 20, 2.0, 3), ("rnbp", 16, 2.0, 1), ("srbp", 12, 2.0, 5)):
    r = po.run(po.Graph.ising(ref, n, c, seed), po.make_config(kind, low_p=0.5, max_iterations=100000, seed=seed))
    out[kind] = {"converged": r.converged, "iterations": r.iterations, "beliefs": r.beliefs.tolist()}
try:
    out["shim_calls"] = int(ctypes.CDLL(%r).bpsched_cuda_shim_calls())
except OSError:
    out["shim_calls"] = None
print(json.dumps(out))
"""


def _run(preload):
    env = dict(os.environ)
    if preload:
        env["LD_PRELOAD"] = SHIM
    p = subprocess.run([sys.executable, "-c", PROG % (ROOT, SHIM)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.skipif(not os.path.exists(SHIM), reason="shim not built (make -C oracle shim)")
def test_preloaded_shim_routes_reference_callers_to_the_device():
    cpu = _run(False)
    gpu = _run(True)
    assert gpu["shim_calls"] == 3  # every bpsched::run call of the reference went through the shim
    for kind in ("lbp", "rnbp"):
        assert gpu[kind]["converged"] and cpu[kind]["converged"], kind
        assert np.max(np.abs(np.array(gpu[kind]["beliefs"]) - np.array(cpu[kind]["beliefs"]))) <= 1e-4, kind
    assert abs(gpu["lbp"]["iterations"] - cpu["lbp"]["iterations"]) <= 1
    # serial RBP stays on the host: bitwise the reference's result
    assert gpu["srbp"] == cpu["srbp"]
