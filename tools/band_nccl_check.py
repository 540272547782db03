"""Band LBP / RnBP through NcclExchange/NcclComm under torchrun; rank 0 checks
the owned beliefs against the one-GPU run (prints OK / FAIL)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1909_11469_b200 as bp  # noqa: E402
from paper_1909_11469_b200 import parallel as par  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
n, c, seed, iters = 24, 2.0, 3, 15
ok = True
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.lbp, max_iterations=iters)
band = par.BandLBP(n, c, seed, rank, world, cfg, local)
st = par.run_band_lbp(band, par.NcclExchange(rank, world), iters)
full = bp.run(bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed), device=local), cfg)
ok &= st.iterations == full.iterations
ok &= bool(np.array_equal(band.owned_beliefs(), full.beliefs.values.reshape(n, n, 2)[band.info.row0:band.info.row1]))
cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5, max_iterations=300, seed=seed)
bands = [par.BandRnBP(n, c, seed, rank, world, cfg, local)]
st = par.run_band_rnbp(bands, par.NcclComm(rank, world), cfg.max_iterations)
full = bp.run(bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed), device=local), cfg)
ok &= st.iterations == full.iterations and st.messages_updated_total == full.messages_updated_total
ok &= bool(np.array_equal(bands[0].owned_beliefs(), full.beliefs.values.reshape(n, n, 2)[bands[0].info.row0:bands[0].info.row1]))
# the C++ driver (csrc/partition.cu): the engine enqueues ncclSend/Recv +
# ncclAllReduce on the band stream itself; torch only broadcasts the NCCL id
obj = [par.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
comm = par.BandComm.nccl(obj[0], rank, world, local)
for kind, kw, iters in (("lbp", {}, 15), ("rnbp", dict(low_p=0.5, seed=seed), 300)):
    cfg = bp.SchedulerConfig(kind=bp.SchedulerKind.from_string(kind), max_iterations=iters, **kw)
    band = par.Band(cfg, rank, world, local, n=n, c=c, seed=seed)
    st = par.run_bands([band], comm)
    full = bp.run(bp.generate_ising(bp.IsingParams(n=n, c=c, seed=seed), device=local), cfg)
    ok &= st.iterations == full.iterations and st.converged == full.converged
    ok &= bool(np.array_equal(band.owned_beliefs(),
                              full.beliefs.values.reshape(n, n, 2)[band.info.row0:band.info.row1]))
    print(f"rank {rank} C++ NCCL band {kind}: iterations {st.iterations} / {full.iterations}", flush=True)
del comm
t = torch.tensor([1 if ok else 0], device="cuda")
dist.all_reduce(t, op=dist.ReduceOp.MIN)
if rank == 0:
    print("OK" if int(t.item()) == 1 else "FAIL")
dist.destroy_process_group()
