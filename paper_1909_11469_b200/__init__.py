"""B200-native belief-propagation message-scheduling engine (arXiv 1909.11469).

Python mirror of the reference ``bpsched`` API for the scheduling hot path
(/root/reference/proj/core/include/bpsched/{mrf,schedulers,generators}.hpp),
bound through ctypes to the C ABI in ``include/bp_cuda.h`` implemented by the
in-tree ``libbp_b200.so`` (hand-written sm_100a kernels).  There is no CPU
fallback: every compute call runs on the GPU, and importing this package
fails loudly when the extension has not been built.

    import paper_1909_11469_b200 as bp
    g = bp.generate_ising(bp.IsingParams(n=100, c=2.5, seed=500))
    r = bp.run(g, bp.SchedulerConfig(kind=bp.SchedulerKind.rnbp, low_p=0.5))
    r.converged, r.iterations, r.beliefs.at(0)
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

__all__ = [
    "SchedulerKind", "SchedulerConfig", "IterationRecord", "RunResult", "BeliefTable", "PairwiseMRF",
    "EdgeSpec", "IsingParams", "ChainParams", "build_graph", "generate_ising", "generate_chain",
    "generate_potts", "generate_er", "generate_ising_arrays", "run", "run_ex", "EngineState", "select_parallelism",
    "Error", "ModelError", "NumericError", "UnsupportedError", "CudaError", "library_path",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("BPB_LIB") or os.path.join(_HERE, "libbp_b200.so")  # BPB_LIB: A/B builds


def library_path() -> str:
    return _LIB_PATH


# --------------------------------------------------------------------------
# errors (errors.hpp:10-38); std::invalid_argument -> ValueError

class Error(RuntimeError):
    """bpsched::error"""


class ModelError(Error):
    """bpsched::model_error"""


class NumericError(Error):
    """bpsched::numeric_error"""


class UnsupportedError(Error):
    pass


class ParseError(Error):
    """bpsched::parse_error (errors.hpp:29-38): the message starts with "line N: "."""

    @property
    def line(self) -> int:
        return int(str(self).split(":", 1)[0].split()[1])


class CudaError(Error):
    pass


_CODES = {1: ValueError, 2: ModelError, 3: NumericError, 4: CudaError, 5: CudaError, 6: MemoryError,
          7: UnsupportedError, 8: ParseError}


# --------------------------------------------------------------------------
# ctypes structures (bp_cuda.h)

class _Desc(C.Structure):
    _fields_ = [("num_vertices", C.c_uint32), ("num_edges", C.c_uint32),
                ("cardinalities", C.c_void_p), ("unary_values", C.c_void_p),
                ("edge_endpoints", C.c_void_p), ("pairwise_values", C.c_void_p)]


class _DevOpts(C.Structure):
    _fields_ = [("device", C.c_int32), ("flags", C.c_uint32)]


class _Config(C.Structure):
    _fields_ = [("kind", C.c_int32), ("splash_depth", C.c_uint32), ("epsilon", C.c_double),
                ("p", C.c_double), ("low_p", C.c_double), ("high_p", C.c_double),
                ("edge_ratio_threshold", C.c_double), ("max_iterations", C.c_uint64),
                ("time_limit", C.c_double), ("seed", C.c_uint64), ("worker_count", C.c_uint32),
                ("_pad", C.c_uint32)]


class _Record(C.Structure):
    _fields_ = [("iteration", C.c_uint64), ("frontier_size", C.c_uint64), ("unconverged", C.c_uint32),
                ("_pad", C.c_uint32), ("elapsed_seconds", C.c_double)]


class _Result(C.Structure):
    _fields_ = [("converged", C.c_int32), ("stopped", C.c_int32), ("iterations", C.c_uint64),
                ("wall_time", C.c_double), ("messages_updated_total", C.c_uint64),
                ("trace_len", C.c_uint64), ("device_ms", C.c_double),
                ("message_evaluations", C.c_uint64), ("gpu_launches", C.c_uint64),
                ("vertex_visits", C.c_uint64), ("splashes", C.c_uint64), ("splash_rounds", C.c_uint64),
                ("persist_iterations", C.c_uint64), ("fused_iterations", C.c_uint64)]


class _Info(C.Structure):
    _fields_ = [("num_vertices", C.c_uint32), ("num_edges", C.c_uint32), ("max_cardinality", C.c_uint32),
                ("state_stride", C.c_uint32), ("device_bytes", C.c_uint64), ("device", C.c_int32),
                ("layout", C.c_uint32), ("message_values", C.c_uint64)]


class KernelStats(C.Structure):
    _fields_ = [("ms", C.c_double * 9), ("launches", C.c_uint64 * 9), ("bytes", C.c_uint64 * 9)]

    CLASSES = ("update", "select", "topk", "splash", "init", "beliefs", "other", "persist", "fused")

    def as_dict(self):
        return {n: {"ms": self.ms[i], "launches": int(self.launches[i]), "bytes": int(self.bytes[i])}
                for i, n in enumerate(self.CLASSES)}


class _RunOpts(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("batch", C.c_uint32), ("stats", C.POINTER(KernelStats)),
                ("beliefs_device", C.c_void_p), ("messages_host", C.c_void_p)]


RUN_KERNEL_TIMING = 1
RUN_NO_GRAPHS = 2
RUN_NO_BELIEFS = 4
RUN_NO_PERSIST = 8
RUN_LBP_TMA = 16
RUN_LBP_TILES = 32
RUN_LBP_VERTEX = 64
RUN_NO_FUSED = 128
RUN_FUSED_TMA = 256
RUN_FUSED_REGS = 512
LBP_KERNELS = {0: "vertex", 1: "tiles", 2: "tma", 3: "qlanes"}  # BP_LBP_KERNEL_*
GRAPH_TRUSTED = 1


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"{_LIB_PATH} is missing: build the CUDA extension first (python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(_LIB_PATH)
    P = C.c_void_p
    sig = {
        "bp_last_error": (C.c_char_p, []),
        "bp_abi_version": (C.c_int, []),
        "bp_graph_create": (C.c_int, [C.POINTER(_Desc), C.POINTER(_DevOpts), C.POINTER(P)]),
        "bp_graph_generate_ising": (C.c_int, [C.c_uint32, C.c_double, C.c_uint64, C.POINTER(_DevOpts), C.POINTER(P)]),
        "bp_graph_generate_chain": (C.c_int, [C.c_uint32, C.c_double, C.c_uint64, C.POINTER(_DevOpts), C.POINTER(P)]),
        "bp_graph_generate_potts": (C.c_int, [C.c_uint32, C.c_uint32, C.c_double, C.c_uint64, C.POINTER(_DevOpts),
                                              C.POINTER(P)]),
        "bp_graph_generate_er": (C.c_int, [C.c_uint32, C.c_uint32, C.c_double, C.c_uint64, C.POINTER(_DevOpts),
                                           C.POINTER(P)]),
        "bp_graph_destroy": (None, [P]),
        "bp_generate_ising_arrays": (C.c_int, [C.c_uint32, C.c_double, C.c_uint64, P, P, P, P]),
        "bp_generate_er_arrays": (C.c_int, [C.c_uint32, C.c_uint32, C.c_double, C.c_uint64, P, P, P, P]),
        "bp_pgm_parse": (C.c_int, [C.c_char_p, C.c_uint64, P]),
        "bp_pgm_info": (C.c_int, [P, P, P, P, P]),
        "bp_pgm_arrays": (C.c_int, [P, P, P, P, P]),
        "bp_pgm_destroy": (None, [P]),
        "bp_graph_create_pgm": (C.c_int, [C.c_char_p, C.c_uint64, P, P]),
        "bp_graph_info_get": (C.c_int, [P, C.POINTER(_Info)]),
        "bp_run": (C.c_int, [P, C.POINTER(_Config), C.POINTER(_Result), P, P, C.c_uint64]),
        "bp_run_ex": (C.c_int, [P, C.POINTER(_Config), C.POINTER(_RunOpts), C.POINTER(_Result), P, P, C.c_uint64]),
        "bp_validate_config": (C.c_int, [C.POINTER(_Config)]),
        "bp_select_parallelism": (C.c_double, [C.c_uint32, C.c_uint32, C.POINTER(_Config)]),
        "bp_engine_create": (C.c_int, [P, C.POINTER(_Config), C.POINTER(P)]),
        "bp_engine_destroy": (None, [P]),
        "bp_engine_unconverged": (C.c_int, [P, C.POINTER(C.c_uint32)]),
        "bp_engine_iteration": (C.c_int, [P, C.POINTER(C.c_uint64)]),
        "bp_engine_advance_iteration": (C.c_int, [P]),
        "bp_engine_messages": (C.c_int, [P, P]),
        "bp_engine_candidates": (C.c_int, [P, P]),
        "bp_engine_residuals": (C.c_int, [P, P]),
        "bp_engine_beliefs": (C.c_int, [P, P]),
        "bp_engine_apply_frontier": (C.c_int, [P, P, C.c_uint64]),
        "bp_engine_apply_splashes": (C.c_int, [P, C.c_uint64, P, P, P]),
        "bp_engine_rnbp_frontier": (C.c_int, [P, C.c_double, P, C.POINTER(C.c_uint64)]),
        "bp_engine_rbp_frontier": (C.c_int, [P, C.c_double, P, C.POINTER(C.c_uint64)]),
        "bp_engine_rs_frontier": (C.c_int, [P, C.c_double, C.c_uint32, P, P, P, C.POINTER(C.c_uint64)]),
        "bp_engine_step": (C.c_int, [P, C.POINTER(C.c_uint64)]),
        "bp_engine_lbp_sweep": (C.c_int, [P, C.c_uint32, C.POINTER(C.c_uint32)]),
        "bp_graph_generate_ising_band": (C.c_int, [C.c_uint32, C.c_double, C.c_uint64, C.c_uint32, C.c_uint32,
                                                   C.POINTER(_DevOpts), C.POINTER(P), C.c_void_p]),
        "bp_band_engine_create": (C.c_int, [P, C.POINTER(_Config), C.c_void_p, C.c_void_p, C.POINTER(P)]),
        "bp_band_stream": (C.c_int, [P, C.POINTER(C.c_uint64)]),
        "bp_band_lbp_sweep": (C.c_int, [P]),
        "bp_band_lbp_finish": (C.c_int, [P]),
        "bp_band_status": (C.c_int, [P, C.POINTER(_Result)]),
        "bp_band_rnbp_begin": (C.c_int, [P]),
        "bp_band_rnbp_finish_init": (C.c_int, [P]),
        "bp_band_rnbp_select": (C.c_int, [P, C.c_uint32]),
        "bp_band_rnbp_refresh": (C.c_int, [P]),
        "bp_band_rbp_select": (C.c_int, [P]),
        "bp_band_rs_select": (C.c_int, [P]),
        "bp_band_rnbp_finish": (C.c_int, [P]),
        "bp_band_survivors": (C.c_int, [P, P, C.c_uint64, C.POINTER(C.c_uint64)]),
        "bp_band_rnbp_fallback": (C.c_int, [P, C.c_uint64]),
        "bp_philox_u53": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64]),
        "bp_philox4x32_10_device": (C.c_int, [C.c_int32, C.c_uint64, P, P, P]),
        "bp_philox_u53_device": (C.c_int, [C.c_int32, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()


def _check(rc):
    if rc != 0:
        msg = _lib.bp_last_error().decode(errors="replace")
        raise _CODES.get(rc, Error)(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------------------
# SchedulerKind / SchedulerConfig (schedulers.hpp:21-41)

class SchedulerKind(enum.IntEnum):
    lbp = 0
    serial_rbp = 1
    rbp = 2
    rs = 3
    rnbp = 4

    def __str__(self):  # to_string (schedulers.cpp:58-67)
        return {0: "lbp", 1: "srbp", 2: "rbp", 3: "rs", 4: "rnbp"}[int(self)]

    @staticmethod
    def from_string(name: str) -> Optional["SchedulerKind"]:  # scheduler_from_string (:69-76)
        return {"lbp": SchedulerKind.lbp, "srbp": SchedulerKind.serial_rbp, "serial_rbp": SchedulerKind.serial_rbp,
                "rbp": SchedulerKind.rbp, "rs": SchedulerKind.rs, "rnbp": SchedulerKind.rnbp}.get(name)


@dataclass
class SchedulerConfig:
    kind: SchedulerKind = SchedulerKind.lbp
    epsilon: float = 1e-5
    p: float = 1.0
    splash_depth: int = 2
    low_p: float = 0.7
    high_p: float = 1.0
    edge_ratio_threshold: float = 0.9
    max_iterations: int = 10000
    time_limit: float = 90.0
    seed: int = 0
    worker_count: int = 0

    def _c(self) -> _Config:
        mi = int(self.max_iterations)
        mi = min(mi, 2 ** 64 - 1)
        return _Config(int(self.kind), int(self.splash_depth), float(self.epsilon), float(self.p),
                       float(self.low_p), float(self.high_p), float(self.edge_ratio_threshold), mi,
                       float(self.time_limit), int(self.seed) & (2 ** 64 - 1), int(self.worker_count), 0)

    def validate(self):
        c = self._c()
        _check(_lib.bp_validate_config(C.byref(c)))


def select_parallelism(prev_unconverged: int, new_unconverged: int, config: SchedulerConfig) -> float:
    c = config._c()
    return float(_lib.bp_select_parallelism(prev_unconverged, new_unconverged, C.byref(c)))


@dataclass
class IterationRecord:
    iteration: int
    frontier_size: int
    unconverged: int
    elapsed_seconds: float


_TRACE_DTYPE = np.dtype([("iteration", np.uint64), ("frontier_size", np.uint64), ("unconverged", np.uint32),
                         ("_pad", np.uint32), ("elapsed_seconds", np.float64)])


class Trace(Sequence):
    """RunResult::trace (schedulers.hpp:40-52): a read-only sequence of
    IterationRecord over the records the run copied out (numpy-backed, so a
    10^4-iteration run does not build 10^4 Python objects up front)."""

    def __init__(self, recs: np.ndarray):
        self._r = recs

    def __len__(self):
        return int(self._r.shape[0])

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(len(self)))]
        x = self._r[k]
        return IterationRecord(int(x["iteration"]), int(x["frontier_size"]), int(x["unconverged"]),
                               float(x["elapsed_seconds"]))

    def column(self, name: str) -> np.ndarray:
        """one field of every record as an array (iteration, frontier_size, ...)"""
        return self._r[name]

    def __eq__(self, other):
        return list(self) == list(other)


class BeliefTable:
    """BeliefTable (messages.hpp:83-107): per-vertex probability vectors."""

    def __init__(self, values: np.ndarray, offsets):
        self.values = values
        # an array, or (V, q) of a uniform-cardinality graph: offsets built on
        # first use (no reference to the graph, whose device memory the table
        # must not keep alive)
        self._offsets = offsets

    @property
    def offsets(self) -> np.ndarray:
        if not isinstance(self._offsets, np.ndarray):
            V, q = self._offsets
            self._offsets = np.arange(V + 1, dtype=np.int64) * q
        return self._offsets

    def num_vertices(self) -> int:
        return len(self.offsets) - 1

    def at(self, v: int) -> np.ndarray:
        return self.values[self.offsets[v]:self.offsets[v + 1]]


@dataclass
class RunResult:
    converged: bool
    iterations: int
    wall_time: float
    messages_updated_total: int
    beliefs: Optional[BeliefTable]
    trace: list = field(repr=False)
    device_ms: float = 0.0
    message_evaluations: int = 0
    gpu_launches: int = 0
    vertex_visits: int = 0
    kernel_stats: Optional[dict] = None
    splashes: int = 0
    splash_rounds: int = 0
    persist_iterations: int = 0
    fused_iterations: int = 0
    messages: Optional[np.ndarray] = field(default=None, repr=False)

    def trace_signature(self) -> str:
        """tests/support/test_helpers.hpp:158-166"""
        s = ("C" if self.converged else "N") + f":{self.iterations}:{self.messages_updated_total}"
        for r in self.trace:
            s += f";{r.iteration},{r.frontier_size},{r.unconverged}"
        return s


# --------------------------------------------------------------------------
# graphs (mrf.hpp:31-96)

@dataclass
class EdgeSpec:
    i: int
    j: int
    table: Sequence[float]


@dataclass
class IsingParams:
    n: int = 10
    c: float = 2.0
    seed: int = 0


@dataclass
class ChainParams:
    length: int = 100
    c: float = 2.0
    seed: int = 0


class PairwiseMRF:
    """Device-resident pairwise MRF (immutable; shareable across runs)."""

    def __init__(self, handle, cardinalities: Optional[np.ndarray], uniform: bool = False):
        self._h = handle
        info = _Info()
        _check(_lib.bp_graph_info_get(handle, C.byref(info)))
        self.info = info
        # uniform cardinality: the per-vertex arrays are built on first use only
        # (graph construction from host arrays is on the end-to-end path)
        self._uniform = uniform or cardinalities is None
        self._cards = None if cardinalities is None else np.asarray(cardinalities, np.uint32)
        self._boff = None
        if self._uniform:
            self.unary_size = int(info.num_vertices) * int(info.max_cardinality)
        else:
            self._boff = np.concatenate([[0], np.cumsum(self._cards, dtype=np.int64)])
            self.unary_size = int(self._boff[-1])

    @property
    def cardinalities(self) -> np.ndarray:
        if self._cards is None:
            self._cards = np.full(self.info.num_vertices, self.info.max_cardinality, np.uint32)
        return self._cards

    @property
    def belief_offsets(self) -> np.ndarray:
        if self._boff is None:
            self._boff = np.arange(int(self.info.num_vertices) + 1, dtype=np.int64) * int(self.info.max_cardinality)
        return self._boff

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:  # the module may be torn down first at interpreter exit
            _lib.bp_graph_destroy(h)
            self._h = None

    def num_vertices(self) -> int:
        return int(self.info.num_vertices)

    def num_edges(self) -> int:
        return int(self.info.num_edges)

    def num_directed_edges(self) -> int:
        return 2 * int(self.info.num_edges)

    def cardinality(self, v: int) -> int:
        return int(self.cardinalities[v])

    def max_cardinality(self) -> int:
        return int(self.info.max_cardinality)

    @property
    def device_bytes(self) -> int:
        return int(self.info.device_bytes)

    @property
    def binary(self) -> bool:
        return self.info.layout == 0

    @classmethod
    def from_arrays(cls, cardinalities, unary_values, edge_endpoints, pairwise_values, device: int = -1,
                    trusted: bool = False) -> "PairwiseMRF":
        cards = np.ascontiguousarray(cardinalities, np.uint32)
        un = np.ascontiguousarray(unary_values, np.float64)
        ep = np.ascontiguousarray(np.asarray(edge_endpoints, np.uint32).reshape(-1))
        tb = np.ascontiguousarray(pairwise_values, np.float64)
        if ep.size % 2:
            raise ValueError("edge_endpoints must hold (i, j) pairs")
        uniform = bool(cards.size) and cards.min() == cards.max()
        expected_unary = int(cards[0]) * cards.size if uniform else int(cards.sum(dtype=np.uint64))
        if un.size != expected_unary:
            raise ModelError(f"expected {expected_unary} unary entries, got {un.size}")
        E = ep.size // 2
        if E and uniform:  # uniform cardinality: q^2 entries per table
            q = int(cards[0])
            if tb.size != E * q * q:
                raise ModelError(f"pairwise tables hold {tb.size} entries, expected {E * q * q}")
        elif E:
            i, j = ep[0::2], ep[1::2]
            ok = (i < cards.size) & (j < cards.size)
            sizes = np.where(ok, cards[np.minimum(i, max(cards.size - 1, 0))].astype(np.int64) *
                             cards[np.minimum(j, max(cards.size - 1, 0))].astype(np.int64), 0)
            if tb.size != int(sizes.sum()) and ok.all():
                raise ModelError(f"pairwise tables hold {tb.size} entries, expected {int(sizes.sum())}")
        d = _Desc(cards.size, E, _ptr(cards), _ptr(un), _ptr(ep), _ptr(tb))
        o = _DevOpts(device, GRAPH_TRUSTED if trusted else 0)
        h = C.c_void_p()
        _check(_lib.bp_graph_create(C.byref(d), C.byref(o), C.byref(h)))
        return cls(h, cards, uniform)


def build_graph(cardinalities: Sequence[int], unary_tables: Sequence[Sequence[float]],
                edges: Iterable) -> PairwiseMRF:
    """build_graph (mrf.cpp:25-106): same validation, same ids, device upload."""
    cards = np.asarray(list(cardinalities), np.uint32)
    unary_tables = list(unary_tables)
    if len(unary_tables) != cards.size:
        raise ModelError(f"expected one unary table per vertex, got {len(unary_tables)} for {cards.size} vertices")
    for v, (c, t) in enumerate(zip(cards, unary_tables)):
        if c == 0:
            raise ModelError(f"vertex {v} has cardinality 0")
        if len(t) != c:
            raise ModelError(f"unary table of vertex {v} has {len(t)} entries, expected {c}")
    un = np.concatenate([np.asarray(t, np.float64) for t in unary_tables]) if unary_tables else np.zeros(0)
    ep, tabs = [], []
    for e, spec in enumerate(edges):
        if isinstance(spec, EdgeSpec):
            i, j, t = spec.i, spec.j, spec.table
        else:
            i, j, t = spec
        ep += [i, j]
        if 0 <= i < cards.size and 0 <= j < cards.size and len(t) != int(cards[i]) * int(cards[j]):
            raise ModelError(f"pairwise table of edge ({i}, {j}) has {len(t)} entries, expected "
                             f"{int(cards[i]) * int(cards[j])}")
        tabs.append(np.asarray(t, np.float64))
    tb = np.concatenate(tabs) if tabs else np.zeros(0)
    return PairwiseMRF.from_arrays(cards, un, np.asarray(ep, np.uint32), tb)


def _gen(fn, *args, device=-1, cards=None):
    o = _DevOpts(device, GRAPH_TRUSTED)
    h = C.c_void_p()
    _check(fn(*args, C.byref(o), C.byref(h)))
    return PairwiseMRF(h, cards)


def generate_ising(params: IsingParams, device: int = -1) -> PairwiseMRF:
    """generate_ising (generators.cpp:24-50), bit-identical instance."""
    return _gen(_lib.bp_graph_generate_ising, params.n, params.c, params.seed, device=device)


def generate_ising_arrays(params: IsingParams):
    """generate_ising's build_graph inputs on the host: (cards, unary, endpoints (E,2), tables)."""
    n = params.n
    V, E = n * n, 2 * n * (n - 1) if n else 0
    cards = np.zeros(max(V, 1), np.uint32)
    un = np.zeros(max(2 * V, 1))
    ep = np.zeros(max(2 * E, 2), np.uint32)
    tb = np.zeros(max(4 * E, 1))
    _check(_lib.bp_generate_ising_arrays(n, params.c, params.seed, _ptr(cards), _ptr(un), _ptr(ep), _ptr(tb)))
    return cards[:V], un[: 2 * V], ep[: 2 * E].reshape(E, 2), tb[: 4 * E]


def parse_model_arrays(text):
    """parse_model (model_io.cpp:98-150) up to build_graph: the reference's text
    model as build_graph's input arrays (cards, unary, endpoints (E, 2), tables),
    parsed on the host pool; ParseError as the reference's parse_error."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    _check(_lib.bp_pgm_parse(data, len(data), C.byref(h)))
    try:
        V, E, nu, nt = C.c_uint32(), C.c_uint32(), C.c_uint64(), C.c_uint64()
        _check(_lib.bp_pgm_info(h, C.byref(V), C.byref(E), C.byref(nu), C.byref(nt)))
        cards = np.zeros(max(V.value, 1), np.uint32)
        un = np.zeros(max(nu.value, 1))
        ep = np.zeros(max(2 * E.value, 2), np.uint32)
        tb = np.zeros(max(nt.value, 1))
        _check(_lib.bp_pgm_arrays(h, _ptr(cards), _ptr(un), _ptr(ep), _ptr(tb)))
    finally:
        _lib.bp_pgm_destroy(h)
    return cards[: V.value], un[: nu.value], ep[: 2 * E.value].reshape(E.value, 2), tb[: nt.value]


def parse_model(text, device: int = -1) -> "PairwiseMRF":
    """parse_model (model_io.cpp:98-150): the text model on the device
    (the arrays of parse_model_arrays through bp_graph_create)."""
    return PairwiseMRF.from_arrays(*parse_model_arrays(text), device=device)


def generate_er_arrays(n: int, m: int, c: float, seed: int):
    """generate_er's instance as build_graph inputs on the host: (cards, unary, endpoints (m,2), tables)."""
    cards = np.zeros(max(n, 1), np.uint32)
    un = np.zeros(max(2 * n, 1))
    ep = np.zeros(max(2 * m, 2), np.uint32)
    tb = np.zeros(max(4 * m, 1))
    _check(_lib.bp_generate_er_arrays(n, m, c, seed, _ptr(cards), _ptr(un), _ptr(ep), _ptr(tb)))
    return cards[:n], un[: 2 * n], ep[: 2 * m].reshape(m, 2), tb[: 4 * m]


def generate_chain(params: ChainParams, device: int = -1) -> PairwiseMRF:
    """generate_chain (generators.cpp:52-71), bit-identical instance."""
    return _gen(_lib.bp_graph_generate_chain, params.length, params.c, params.seed, device=device)


def generate_potts(n: int, q: int, c: float, seed: int, device: int = -1) -> PairwiseMRF:
    """Potts n x n grid, q states."""
    return _gen(_lib.bp_graph_generate_potts, n, q, c, seed, device=device)


def generate_er(n: int, m: int, c: float, seed: int, device: int = -1) -> PairwiseMRF:
    """Erdos-Renyi G(n, m), binary Ising-style potentials."""
    return _gen(_lib.bp_graph_generate_er, n, m, c, seed, device=device)


# --------------------------------------------------------------------------
# run (schedulers.cpp:293-353)

def run_ex(graph: PairwiseMRF, config: SchedulerConfig, flags: int = 0, batch: int = 0, beliefs: bool = True,
           trace_cap: Optional[int] = None, kernel_timing: bool = False, beliefs_device_ptr: int = 0,
           messages: bool = False) -> RunResult:
    """bp_run_ex.  messages=True also returns the live messages at the end of
    the run (RunResult.messages, fp64 probabilities in MessageStore order)."""
    c = config._c()
    msgs = np.empty(max(int(graph.info.message_values), 1)) if messages else None
    nb = graph.unary_size
    bel = np.empty(max(nb, 1)) if beliefs and not beliefs_device_ptr else None  # filled by bp_run_ex
    if trace_cap is None:
        trace_cap = int(min(config.max_iterations, 1 << 20)) + 1
    tr = (_Record * max(trace_cap, 1))()
    res = _Result()
    stats = KernelStats()
    fl = flags | (RUN_KERNEL_TIMING if kernel_timing else 0) | (0 if beliefs else RUN_NO_BELIEFS)
    opts = _RunOpts(fl, batch, C.pointer(stats), beliefs_device_ptr or None, _ptr(msgs))
    _check(_lib.bp_run_ex(graph._h, C.byref(c), C.byref(opts), C.byref(res), _ptr(bel), C.cast(tr, C.c_void_p),
                          trace_cap))
    n = min(int(res.trace_len), trace_cap)
    trace = Trace(np.frombuffer(tr, dtype=_TRACE_DTYPE, count=n).copy())
    boff = graph._boff if graph._boff is not None else (int(graph.info.num_vertices), int(graph.info.max_cardinality))
    bt = BeliefTable(bel[:nb], boff) if bel is not None else None
    return RunResult(bool(res.converged), int(res.iterations), float(res.wall_time),
                     int(res.messages_updated_total), bt, trace, float(res.device_ms),
                     int(res.message_evaluations), int(res.gpu_launches), int(res.vertex_visits),
                     stats.as_dict() if kernel_timing else None, int(res.splashes), int(res.splash_rounds),
                     int(res.persist_iterations), int(res.fused_iterations),
                     msgs[: int(graph.info.message_values)] if msgs is not None else None)


def run(graph: PairwiseMRF, config: SchedulerConfig) -> RunResult:
    """bpsched::run: to convergence or cap; caps give converged=False, not an error."""
    return run_ex(graph, config)


# --------------------------------------------------------------------------
# the device random stream (diagnostics for known-answer tests)

def philox4x32_10_device(ctr, key, device: int = -1) -> np.ndarray:
    """The device's Philox4x32-10 on counters (n, 4) / keys (n, 2) -> (n, 4) uint32."""
    ctr = np.ascontiguousarray(ctr, np.uint32).reshape(-1, 4)
    key = np.ascontiguousarray(key, np.uint32).reshape(-1, 2)
    out = np.zeros_like(ctr)
    _check(_lib.bp_philox4x32_10_device(device, ctr.shape[0], _ptr(ctr), _ptr(key), _ptr(out)))
    return out


def philox_u53_device(seed: int, iteration: int, attempt: int, d, device: int = -1) -> np.ndarray:
    """53-bit RnBP draws of directed edges d in (seed, iteration, attempt), on the device."""
    d = np.ascontiguousarray(d, np.uint64)
    out = np.zeros_like(d)
    _check(_lib.bp_philox_u53_device(device, seed, iteration, attempt, d.size, _ptr(d), _ptr(out)))
    return out


def philox_u53(seed: int, iteration: int, attempt: int, d: int) -> int:
    """Host restatement of the same draw (bp_philox_u53; the band fallback)."""
    return int(_lib.bp_philox_u53(seed, iteration, attempt, d))


# EngineState + per-phase API (schedulers.hpp:61-151), for lockstep parity

class EngineState:
    def __init__(self, graph: PairwiseMRF, config: SchedulerConfig):
        self.graph = graph
        self.config = config
        self._cfg = config._c()
        h = C.c_void_p()
        _check(_lib.bp_engine_create(graph._h, C.byref(self._cfg), C.byref(h)))
        self._h = h
        self.D = graph.num_directed_edges()
        # message offsets: length card(target(d)) per directed edge
        self._moff = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.bp_engine_destroy(h)
            self._h = None

    def _total(self):
        if self._moff is None:
            if self.graph.binary:
                self._moff = np.arange(self.D + 1, dtype=np.int64) * 2
            else:
                raise RuntimeError("set_endpoints() required for generic graphs")
        return int(self._moff[-1])

    def set_endpoints(self, endpoints: np.ndarray):
        ep = np.asarray(endpoints, np.int64).reshape(-1, 2)
        tgt = np.empty(2 * ep.shape[0], np.int64)
        tgt[0::2] = ep[:, 1]
        tgt[1::2] = ep[:, 0]
        lens = self.graph.cardinalities[tgt].astype(np.int64)
        self._moff = np.concatenate([[0], np.cumsum(lens)])

    def unconverged_count(self) -> int:
        n = C.c_uint32()
        _check(_lib.bp_engine_unconverged(self._h, C.byref(n)))
        return int(n.value)

    def iteration(self) -> int:
        n = C.c_uint64()
        _check(_lib.bp_engine_iteration(self._h, C.byref(n)))
        return int(n.value)

    def messages(self) -> np.ndarray:
        out = np.zeros(max(self._total(), 1))
        _check(_lib.bp_engine_messages(self._h, _ptr(out)))
        return out[: self._total()]

    def candidates(self) -> np.ndarray:
        out = np.zeros(max(self._total(), 1))
        _check(_lib.bp_engine_candidates(self._h, _ptr(out)))
        return out[: self._total()]

    def residuals(self) -> np.ndarray:
        out = np.zeros(max(self.D, 1))
        _check(_lib.bp_engine_residuals(self._h, _ptr(out)))
        return out[: self.D]

    def beliefs(self) -> np.ndarray:
        nb = int(self.graph.belief_offsets[-1])
        out = np.zeros(max(nb, 1))
        _check(_lib.bp_engine_beliefs(self._h, _ptr(out)))
        return out[:nb]

    def apply_frontier(self, frontier) -> None:
        f = np.ascontiguousarray(frontier, np.uint32)
        _check(_lib.bp_engine_apply_frontier(self._h, _ptr(f) if f.size else None, f.size))

    def rnbp_frontier(self, p: float) -> np.ndarray:
        out = np.zeros(max(self.D, 1), np.uint32)
        n = C.c_uint64()
        _check(_lib.bp_engine_rnbp_frontier(self._h, p, _ptr(out), C.byref(n)))
        return out[: n.value].copy()

    def rbp_frontier(self, p: float) -> np.ndarray:
        out = np.zeros(max(self.D, 1), np.uint32)
        n = C.c_uint64()
        _check(_lib.bp_engine_rbp_frontier(self._h, p, _ptr(out), C.byref(n)))
        return out[: n.value].copy()

    def rs_frontier(self, p: float, h: int):
        V = self.graph.num_vertices()
        roots = np.zeros(max(V, 1), np.uint32)
        eoff = np.zeros(V + 1, np.uint64)
        edges = np.zeros(max(self.D, 1), np.uint32)
        n = C.c_uint64()
        _check(_lib.bp_engine_rs_frontier(self._h, p, h, _ptr(roots), _ptr(eoff), _ptr(edges), C.byref(n)))
        k = n.value
        return roots[:k].copy(), eoff[: k + 1].copy(), edges[: int(eoff[k])].copy()

    def apply_splashes(self, roots, eoff, edges) -> None:
        roots = np.ascontiguousarray(roots, np.uint32)
        eoff = np.ascontiguousarray(eoff, np.uint64)
        edges = np.ascontiguousarray(edges, np.uint32)
        _check(_lib.bp_engine_apply_splashes(self._h, roots.size, _ptr(roots), _ptr(eoff), _ptr(edges)))

    def advance_iteration(self) -> None:
        """EngineState::advance_iteration (schedulers.hpp:75): the Philox draws of
        the next rnbp_frontier use the next iteration's keys."""
        _check(_lib.bp_engine_advance_iteration(self._h))

    def step(self) -> int:
        n = C.c_uint64()
        _check(_lib.bp_engine_step(self._h, C.byref(n)))
        return int(n.value)

    def lbp_sweep(self, kernel: str = "auto") -> str:
        """One fused LBP sweep with the production kernel (bp_engine_lbp_sweep):
        afterwards messages() = m_t, candidates() = f(m_t), unconverged_count()
        = #{r(m_t) >= eps}.  kernel: "auto" | "tma" | "tiles" | "vertex"; returns
        the kernel that ran ("vertex", "tiles", "tma" or "qlanes")."""
        flags = {"auto": 0, "tma": RUN_LBP_TMA, "tiles": RUN_LBP_TILES, "vertex": RUN_LBP_VERTEX}[kernel]
        k = C.c_uint32()
        _check(_lib.bp_engine_lbp_sweep(self._h, flags, C.byref(k)))
        return LBP_KERNELS[int(k.value)]
