"""Row-band partition of a lattice across GPUs.

One process per GPU.  Rank g owns rows [g*n/P, (g+1)*n/P) of the
generate_ising(n, c, seed) grid (generators.cpp:24-50) and every message whose
source it owns; its band adds one ghost row per neighbouring band.  One LBP
iteration (schedulers.cpp:301-347 with the LBP frontier) is

    bp_band_lbp_sweep    sweep of the band on the device; boundary messages
                         -> send_up / send_down; local unconverged count and
                         time-limit vote -> count[0..1]
    exchange             send_up -> rank g-1 (its recv_down), send_down ->
                         rank g+1 (its recv_up); all-reduce(sum) of count
    bp_band_lbp_finish   ghost messages <- recv_*; the loop control of run()
                         on the GLOBAL count

all enqueued on the band's own CUDA stream (torch.cuda.ExternalStream), so
there is no host synchronisation inside the loop; the host polls the stop flag
every `check_every` iterations (iterations after a stop are no-ops on the
device).  Owned messages are bitwise identical to the unpartitioned run, so
results do not depend on the GPU count (the determinism contract of
thread_pool.hpp:13-16, restated for GPUs).

The transport is torch.distributed: NCCL over NVLink between GPUs, gloo on
CPU for the host-logic tests (tests/test_parallel_cpu.py), or `LocalExchange`
for several bands inside one process on one device (parity tests).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import (_Config, _DevOpts, _Result, _check, _lib, GRAPH_TRUSTED, PairwiseMRF, SchedulerConfig,
               SchedulerKind)

__all__ = ["band_rows", "owned_directed_edges", "BandInfo", "Band", "BandComm", "nccl_unique_id", "run_bands",
           "BandLBP", "BandRnBP", "BandRBP", "BandRS", "NcclExchange", "LocalExchange", "NcclComm", "LocalComm",
           "run_band_lbp", "run_band_rnbp"]


def band_rows(n: int, part: int, nparts: int):
    """Owned rows [r0, r1) and ghost flags of band `part` (mirrors bp_graph_generate_ising_band)."""
    if nparts < 1 or not 0 <= part < nparts or nparts > n:
        raise ValueError("bad band partition")
    r0, r1 = part * n // nparts, (part + 1) * n // nparts
    return r0, r1, int(part > 0), int(part + 1 < nparts)


def owned_directed_edges(n: int, r0: int, r1: int) -> int:
    """Directed edges whose source lies in rows [r0, r1) of an n x n grid (sum of degrees)."""
    return sum(n * ((r > 0) + (r + 1 < n)) + 2 * (n - 1) for r in range(r0, r1))


class _BandInfoC(C.Structure):
    _fields_ = [("part", C.c_uint32), ("nparts", C.c_uint32), ("row0", C.c_uint32), ("row1", C.c_uint32),
                ("ghost_up", C.c_uint32), ("ghost_down", C.c_uint32), ("local_rows", C.c_uint32),
                ("cols", C.c_uint32), ("owned_directed", C.c_uint64)]


class _HaloC(C.Structure):
    _fields_ = [("send_up", C.c_void_p), ("send_down", C.c_void_p), ("recv_up", C.c_void_p),
                ("recv_down", C.c_void_p), ("count", C.c_void_p)]


@dataclass
class BandInfo:
    part: int
    nparts: int
    row0: int
    row1: int
    ghost_up: int
    ghost_down: int
    local_rows: int
    cols: int
    owned_directed: int


@dataclass
class BandStatus:
    stopped: bool
    converged: bool
    iterations: int
    messages_updated_total: int  # this band's owned messages
    gpu_launches: int


class BandLBP:
    """LBP on one band of the n x n Ising grid, on cuda:`device`."""

    KIND = SchedulerKind.lbp
    NCOUNT = 2  # {unconverged count, time vote}

    def __init__(self, n: int, c: float, seed: int, part: int, nparts: int, config: SchedulerConfig,
                 device: int = 0):
        import torch

        if config.kind != self.KIND:
            raise ValueError(f"{type(self).__name__} needs kind={self.KIND}")
        self.seed = int(config.seed)
        info = _BandInfoC()
        h = C.c_void_p()
        _check(_lib.bp_graph_generate_ising_band(n, c, seed, part, nparts, C.byref(_DevOpts(device, GRAPH_TRUSTED)),
                                                 C.byref(h), C.byref(info)))
        self.graph = PairwiseMRF(h, None)
        self.info = BandInfo(*(getattr(info, f) for f, _ in _BandInfoC._fields_))
        dev = torch.device("cuda", device)
        cols = self.info.cols
        self.send_up = torch.zeros(cols, dtype=torch.float32, device=dev)
        self.send_down = torch.zeros(cols, dtype=torch.float32, device=dev)
        self.recv_up = torch.zeros(cols, dtype=torch.float32, device=dev)
        self.recv_down = torch.zeros(cols, dtype=torch.float32, device=dev)
        self.count = torch.zeros(self.NCOUNT, dtype=torch.int64, device=dev)
        halo = _HaloC(self.send_up.data_ptr(), self.send_down.data_ptr(), self.recv_up.data_ptr(),
                      self.recv_down.data_ptr(), self.count.data_ptr())
        self._cfg = config._c()
        e = C.c_void_p()
        torch.cuda.synchronize(dev)  # buffers initialised before the engine's stream uses them
        _check(_lib.bp_band_engine_create(self.graph._h, C.byref(self._cfg), C.byref(info), C.byref(halo),
                                          C.byref(e)))
        self._e = e
        s = C.c_uint64()
        _check(_lib.bp_band_stream(e, C.byref(s)))
        self.stream = torch.cuda.ExternalStream(s.value, device=dev)

    def __del__(self):
        e = getattr(self, "_e", None)
        if e and _lib is not None:
            _lib.bp_engine_destroy(e)
            self._e = None

    def sweep(self):
        _check(_lib.bp_band_lbp_sweep(self._e))

    def finish(self):
        _check(_lib.bp_band_lbp_finish(self._e))

    def beliefs(self):
        """Beliefs of every band vertex (ghost rows included) from the current messages."""
        import numpy as np

        out = np.zeros(2 * self.graph.num_vertices())
        _check(_lib.bp_engine_beliefs(self._e, out.ctypes.data_as(C.c_void_p)))
        return out.reshape(self.info.local_rows, self.info.cols, 2)

    def owned_beliefs(self):
        g = self.info.ghost_up
        return self.beliefs()[g:g + self.info.row1 - self.info.row0]

    def status(self) -> BandStatus:
        r = _Result()
        _check(_lib.bp_band_status(self._e, C.byref(r)))
        return BandStatus(bool(r.stopped), bool(r.converged), int(r.iterations), int(r.messages_updated_total),
                          int(r.gpu_launches))


class BandRnBP(BandLBP):
    """RnBP on one band (Philox draws keyed by global edge ids, so the run is
    the same for any number of bands)."""

    KIND = SchedulerKind.rnbp
    NCOUNT = 5  # {delta, frontier, survivors, time vote, initial count}

    def begin(self):
        _check(_lib.bp_band_rnbp_begin(self._e))

    def finish_init(self):
        _check(_lib.bp_band_rnbp_finish_init(self._e))

    def select(self, attempt: int = 0):
        _check(_lib.bp_band_rnbp_select(self._e, attempt))

    def refresh(self):
        _check(_lib.bp_band_rnbp_refresh(self._e))

    def finish(self):
        _check(_lib.bp_band_rnbp_finish(self._e))

    def survivors(self):
        import numpy as np

        n = C.c_uint64()
        _check(_lib.bp_band_survivors(self._e, None, 0, C.byref(n)))
        out = np.zeros(max(int(n.value), 1), np.uint64)
        _check(_lib.bp_band_survivors(self._e, out.ctypes.data_as(C.c_void_p), out.size, C.byref(n)))
        return out[: int(n.value)]

    def fallback(self, global_d: int):
        _check(_lib.bp_band_rnbp_fallback(self._e, global_d))


class BandRBP(BandRnBP):
    """RBP on one band with a per-partition local frontier: the band's top
    k = max(1, llround(p * owned directed edges)) residuals."""

    KIND = SchedulerKind.rbp

    def select(self, attempt: int = 0):
        _check(_lib.bp_band_rbp_select(self._e))


class BandRS(BandRnBP):
    """Residual Splash on one band with per-partition local splashes (roots and
    claims on owned vertices, k = max(1, llround(p * owned vertices)))."""

    KIND = SchedulerKind.rs

    def select(self, attempt: int = 0):
        _check(_lib.bp_band_rs_select(self._e))


class NcclComm:
    """Collectives of one band per process (torch.distributed, NCCL between GPUs)."""

    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world
        self._halo = NcclExchange(rank, world)

    def halo(self, bands):
        import torch.distributed as dist

        import torch

        (b,) = bands
        ops = []
        if b.info.ghost_up:
            ops += [dist.P2POp(dist.isend, b.send_up, self.rank - 1), dist.P2POp(dist.irecv, b.recv_up, self.rank - 1)]
        if b.info.ghost_down:
            ops += [dist.P2POp(dist.isend, b.send_down, self.rank + 1),
                    dist.P2POp(dist.irecv, b.recv_down, self.rank + 1)]
        # on the band's (non-blocking) stream: ordered after the select / pack
        # kernels that fill send_*, and before the refresh that reads recv_*
        if ops:
            with torch.cuda.stream(b.stream):
                for w in dist.batch_isend_irecv(ops):
                    w.wait()

    def reduce(self, bands):
        import torch
        import torch.distributed as dist

        with torch.cuda.stream(bands[0].stream):  # after k_part_count_rnbp wrote count
            dist.all_reduce(bands[0].count)

    def gather_lists(self, lists):
        import torch.distributed as dist

        out = [None] * self.world
        dist.all_gather_object(out, [int(x) for x in lists[0]])
        return out


class LocalComm:
    """All bands in one process on one device (tests): the same data movement."""

    def halo(self, bands):
        import torch

        torch.cuda.synchronize()
        for i, b in enumerate(bands):
            if b.info.ghost_up:
                b.recv_up.copy_(bands[i - 1].send_down)
            if b.info.ghost_down:
                b.recv_down.copy_(bands[i + 1].send_up)
        torch.cuda.synchronize()

    def reduce(self, bands):
        import torch

        torch.cuda.synchronize()
        total = sum(b.count.clone() for b in bands)
        for b in bands:
            b.count.copy_(total)
        torch.cuda.synchronize()

    def gather_lists(self, lists):
        return [[int(x) for x in l] for l in lists]


def run_band_rnbp(bands, comm, max_iterations: int) -> BandStatus:
    """The run() loop of RnBP (or RBP, BandRBP) over row bands
    (schedulers.cpp:301-347 with rnbp_frontier :194-216 / rbp_frontier
    :122-126): `bands` are this process's bands (one per GPU with NcclComm, all
    of them with LocalComm)."""
    import torch

    def phase(attempt):
        for b in bands:
            with torch.cuda.stream(b.stream):
                b.select(attempt)
        comm.halo(bands)
        for b in bands:
            with torch.cuda.stream(b.stream):
                b.refresh()
        comm.reduce(bands)

    for b in bands:
        with torch.cuda.stream(b.stream):
            b.begin()
    comm.reduce(bands)
    for b in bands:
        with torch.cuda.stream(b.stream):
            b.finish_init()
    for _ in range(max_iterations + 1):
        st = bands[0].status()
        if st.stopped:
            return st
        phase(0)
        with torch.cuda.stream(bands[0].stream):  # the D2H read is ordered after the all-reduce
            delta, frontier, survivors = (int(x) for x in bands[0].count[:3].tolist())
        rnbp = bands[0].KIND == SchedulerKind.rnbp
        if rnbp and frontier == 0 and survivors > 0:  # retry once, then one survivor (schedulers.cpp:204-214)
            phase(1)
            with torch.cuda.stream(bands[0].stream):
                frontier = int(bands[0].count[1].item())
            if frontier == 0:
                ids = sorted(x for l in comm.gather_lists([b.survivors() for b in bands]) for x in l)
                u = _lib.bp_philox_u53(bands[0].seed, st.iterations, 2, 0) * 2.0 ** -53
                pick = ids[min(len(ids) - 1, int(u * len(ids)))]
                for b in bands:
                    owned = pick in set(int(x) for x in b.survivors())
                    with torch.cuda.stream(b.stream):
                        b.fallback(pick if owned else (1 << 64) - 1)
                comm.halo(bands)
                for b in bands:
                    with torch.cuda.stream(b.stream):
                        b.refresh()
                comm.reduce(bands)
        for b in bands:
            with torch.cuda.stream(b.stream):
                b.finish()
    return bands[0].status()


class NcclExchange:
    """Halo exchange + count all-reduce through torch.distributed (NCCL on GPUs),
    enqueued on the band's stream."""

    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world

    def __call__(self, band: BandLBP):
        import torch.distributed as dist

        ops = []
        if band.info.ghost_up:
            ops += [dist.P2POp(dist.isend, band.send_up, self.rank - 1),
                    dist.P2POp(dist.irecv, band.recv_up, self.rank - 1)]
        if band.info.ghost_down:
            ops += [dist.P2POp(dist.isend, band.send_down, self.rank + 1),
                    dist.P2POp(dist.irecv, band.recv_down, self.rank + 1)]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        dist.all_reduce(band.count)


class LocalExchange:
    """All bands in one process (one device): the same data movement as
    NcclExchange with device copies; host-synchronised (tests only)."""

    def __init__(self, bands):
        self.bands = bands

    def exchange_all(self):
        import torch

        torch.cuda.synchronize()
        bands = self.bands
        for i, b in enumerate(bands):
            if b.info.ghost_up:
                b.recv_up.copy_(bands[i - 1].send_down)
            if b.info.ghost_down:
                b.recv_down.copy_(bands[i + 1].send_up)
        total = sum(b.count.clone() for b in bands)
        for b in bands:
            b.count.copy_(total)
        torch.cuda.synchronize()


def run_band_lbp(band: BandLBP, exchange, max_iterations: int, check_every: int = 16) -> BandStatus:
    """The run() loop of one band (all ranks call it with the same arguments)."""
    import torch

    with torch.cuda.stream(band.stream):
        for it in range(max_iterations + 1):  # sweep 0 computes r(m_0) (ResidualTracker ctor)
            band.sweep()
            exchange(band)
            band.finish()
            if it % check_every == check_every - 1:
                st = band.status()
                if st.stopped:
                    return st
    return band.status()


# ---------------------------------------------------------------------------
# The C++ driver (csrc/partition.cu): the run() loop of a band with the halo
# exchange and the counter all-reduce enqueued on the band's stream by the
# engine itself (NCCL between ranks), no Python inside the loop.

def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype, f.argtypes = res, args
    return f


_P = C.c_void_p
_create_band = _sig("bp_graph_create_band", C.c_int, [_P, C.c_uint32, C.c_uint32, C.POINTER(_DevOpts), C.POINTER(_P),
                                                      C.POINTER(_BandInfoC)])
_create_owned = _sig("bp_band_engine_create_owned", C.c_int, [_P, C.POINTER(_Config), C.POINTER(_BandInfoC),
                                                              C.POINTER(_P)])
_unique_id = _sig("bp_nccl_unique_id", C.c_int, [_P])
_comm_nccl = _sig("bp_band_comm_create_nccl", C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_int32, C.POINTER(_P)])
_comm_local = _sig("bp_band_comm_create_local", C.c_int, [C.POINTER(_P)])
_comm_destroy = _sig("bp_band_comm_destroy", None, [_P])
_band_run = _sig("bp_band_run", C.c_int, [_P, C.c_uint32, _P, C.POINTER(_Result)])


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId on this rank (128 bytes; broadcast it to the other ranks)."""
    buf = (C.c_uint8 * 128)()
    _check(_unique_id(buf))
    return bytes(buf)


class BandComm:
    """The exchange of the C++ band loop: `nccl(id, rank, nranks, device)` links
    one band per rank; `local()` drives every band of the partition in this
    process (host-staged copies; one GPU in the tests)."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def nccl(cls, uid: bytes, rank: int, nranks: int, device: int = -1) -> "BandComm":
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(_comm_nccl(buf, rank, nranks, device, C.byref(h)))
        return cls(h)

    @classmethod
    def local(cls) -> "BandComm":
        h = C.c_void_p()
        _check(_comm_local(C.byref(h)))
        return cls(h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _comm_destroy(h)
            self._h = None


class Band:
    """One band of a row partition with engine-owned halo buffers, driven by
    run_bands.  Either band `part` of generate_ising(n, c, seed), or of any
    binary Ising lattice given as build_graph arrays (generate_ising's edge
    numbering, any rows x cols)."""

    def __init__(self, config: SchedulerConfig, part: int, nparts: int, device: int = 0, *, n: int = 0,
                 c: float = 0.0, seed: int = 0, arrays=None):
        import numpy as np

        info = _BandInfoC()
        h = C.c_void_p()
        opts = _DevOpts(device, GRAPH_TRUSTED)
        if arrays is None:
            _check(_lib.bp_graph_generate_ising_band(n, c, seed, part, nparts, C.byref(opts), C.byref(h),
                                                     C.byref(info)))
        else:
            from . import _Desc
            cards, un, ep, tb = (np.ascontiguousarray(arrays[0], np.uint32), np.ascontiguousarray(arrays[1], np.float64),
                                 np.ascontiguousarray(np.asarray(arrays[2]).reshape(-1), np.uint32),
                                 np.ascontiguousarray(arrays[3], np.float64))
            d = _Desc(cards.size, ep.size // 2, cards.ctypes.data_as(C.c_void_p), un.ctypes.data_as(C.c_void_p),
                      ep.ctypes.data_as(C.c_void_p), tb.ctypes.data_as(C.c_void_p))
            _check(_create_band(C.byref(d), part, nparts, C.byref(_DevOpts(device, 0)), C.byref(h), C.byref(info)))
        self.graph = PairwiseMRF(h, None)
        self.info = BandInfo(*(getattr(info, f) for f, _ in _BandInfoC._fields_))
        self._cfg = config._c()
        e = C.c_void_p()
        _check(_create_owned(self.graph._h, C.byref(self._cfg), C.byref(info), C.byref(e)))
        self._e = e

    def __del__(self):
        e = getattr(self, "_e", None)
        if e and _lib is not None:
            _lib.bp_engine_destroy(e)
            self._e = None

    beliefs = BandLBP.beliefs
    owned_beliefs = BandLBP.owned_beliefs
    status = BandLBP.status


class _PartInfoC(C.Structure):
    _fields_ = [("part", C.c_uint32), ("nparts", C.c_uint32), ("v0", C.c_uint32), ("v1", C.c_uint32),
                ("ghost_vertices", C.c_uint32), ("local_edges", C.c_uint32), ("peers", C.c_uint32),
                ("_pad", C.c_uint32), ("send_messages", C.c_uint64), ("recv_messages", C.c_uint64),
                ("owned_directed", C.c_uint64)]


@dataclass
class PartInfo:
    part: int
    nparts: int
    v0: int
    v1: int
    ghost_vertices: int
    local_edges: int
    peers: int
    send_messages: int
    recv_messages: int
    owned_directed: int


_create_part = _sig("bp_graph_create_part", C.c_int, [_P, C.c_uint32, C.c_uint32, C.POINTER(_DevOpts), C.POINTER(_P),
                                                      C.POINTER(_PartInfoC)])
_part_engine = _sig("bp_part_engine_create", C.c_int, [_P, C.POINTER(_Config), C.POINTER(_P)])


class Part:
    """One part of a vertex-range partition of ANY binary model given as
    build_graph arrays (random graphs included): vertices [v0, v1) and the
    messages they send, ghosts for the outside neighbours, cut messages
    exchanged with every peer part each iteration.  Driven by run_bands (LBP,
    RnBP); the run is the unpartitioned one for any number of parts."""

    def __init__(self, config: SchedulerConfig, part: int, nparts: int, arrays, device: int = 0,
                 trusted: bool = False):
        import numpy as np

        from . import _Desc
        cards, un, ep, tb = (np.ascontiguousarray(arrays[0], np.uint32), np.ascontiguousarray(arrays[1], np.float64),
                             np.ascontiguousarray(np.asarray(arrays[2]).reshape(-1), np.uint32),
                             np.ascontiguousarray(arrays[3], np.float64))
        d = _Desc(cards.size, ep.size // 2, cards.ctypes.data_as(C.c_void_p), un.ctypes.data_as(C.c_void_p),
                  ep.ctypes.data_as(C.c_void_p), tb.ctypes.data_as(C.c_void_p))
        info = _PartInfoC()
        h = C.c_void_p()
        _check(_create_part(C.byref(d), part, nparts, C.byref(_DevOpts(device, GRAPH_TRUSTED if trusted else 0)),
                            C.byref(h), C.byref(info)))
        self.graph = PairwiseMRF(h, None)
        self.info = PartInfo(*(getattr(info, f) for f, _ in _PartInfoC._fields_ if f != "_pad"))
        self._cfg = config._c()
        e = C.c_void_p()
        _check(_part_engine(self.graph._h, C.byref(self._cfg), C.byref(e)))
        self._e = e

    def __del__(self):
        e = getattr(self, "_e", None)
        if e and _lib is not None:
            _lib.bp_engine_destroy(e)
            self._e = None

    def owned_beliefs(self):
        """Beliefs (v1 - v0, 2) of the owned vertices, global order."""
        import numpy as np

        out = np.zeros(2 * self.graph.num_vertices())
        _check(_lib.bp_engine_beliefs(self._e, out.ctypes.data_as(C.c_void_p)))
        return out.reshape(-1, 2)[: self.info.v1 - self.info.v0]

    status = BandLBP.status


def run_bands(bands, comm: BandComm) -> BandStatus:
    """The run() loop over row bands in C++ (bp_band_run): NCCL -- this rank's
    band; local -- every band of the partition, parts 0..P-1."""
    arr = (C.c_void_p * len(bands))(*[b._e.value for b in bands])
    r = _Result()
    _check(_band_run(arr, len(bands), comm._h, C.byref(r)))
    return BandStatus(bool(r.stopped), bool(r.converged), int(r.iterations), int(r.messages_updated_total),
                      int(r.gpu_launches))
