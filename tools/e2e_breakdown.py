"""Where the e2e step's time goes: graph build stages (BPB_DEBUG_BUILD), run,
beliefs D2H; plus pageable vs pinned H2D bandwidth of the same 100 MB."""
import os
import sys
import time

os.environ["BPB_DEBUG_BUILD"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1909_11469_b200 as bp  # noqa: E402

torch.cuda.set_device(0)
arrs = {s: bp.generate_ising_arrays(bp.IsingParams(n=1000, c=2.5, seed=s)) for s in range(6)}
cfg = lambda s, it=20: bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=it,
                                          time_limit=1e9, seed=s)
bp.run(bp.PairwiseMRF.from_arrays(*arrs[0]), cfg(0, 2))
for s in range(6):
    t0 = time.perf_counter()
    g = bp.PairwiseMRF.from_arrays(*arrs[s])
    t1 = time.perf_counter()
    r = bp.run(g, cfg(s))
    t2 = time.perf_counter()
    _ = float(r.beliefs.values[-1])
    t3 = time.perf_counter()
    print(f"seed {s}: graph {1e3*(t1-t0):6.1f} run {1e3*(t2-t1):6.1f} (device {r.device_ms:6.2f}) "
          f"sum {1e3*(t3-t2):4.1f}", file=sys.stderr, flush=True)
    del g
tb = arrs[0][3]
dev = torch.empty(tb.size, dtype=torch.float64, device="cuda")
for kind in ("pageable", "pinned"):
    src = torch.from_numpy(tb) if kind == "pageable" else torch.from_numpy(tb).pin_memory()
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        dev.copy_(src, non_blocking=(kind == "pinned")); torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"H2D {kind}: {tb.nbytes/1e6:.0f} MB in {dt*1e3:.2f} ms = {tb.nbytes/dt/1e9:.1f} GB/s", file=sys.stderr)
t0 = time.perf_counter(); x = torch.empty(tb.size, dtype=torch.float64).pin_memory(); t1 = time.perf_counter()
print(f"pin_memory alloc 64MB {1e3*(t1-t0):.1f} ms; nproc {os.cpu_count()}", file=sys.stderr)
a = np.empty_like(tb); t0 = time.perf_counter(); np.copyto(a, tb); t1 = time.perf_counter()
print(f"host memcpy 64MB 1 thread {1e3*(t1-t0):.1f} ms", file=sys.stderr)
import threading
buf = np.ones(64 << 20 >> 3)
for nt in (1, 4, 8, 16):
    parts = np.array_split(buf, nt)
    ths = [threading.Thread(target=lambda p=p: p.sum()) for p in parts]
    t0 = time.perf_counter()
    for t in ths: t.start()
    for t in ths: t.join()
    dt = time.perf_counter() - t0
    print(f"host read 64MB, {nt} threads: {dt*1e3:.2f} ms = {buf.nbytes/dt/1e9:.1f} GB/s", file=sys.stderr)
g = bp.PairwiseMRF.from_arrays(*arrs[1])
for it in range(3):
    r = bp.run(g, cfg(1))
    print(f"same graph back-to-back run {it}: device {r.device_ms:.2f} ms", file=sys.stderr)
