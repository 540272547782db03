"""TEST INFRASTRUCTURE ONLY -- ctypes access to the CPU oracles.

Two interchangeable backends with one API:

* ``load("orc")`` -> ``oracle/liboracle.so``: the plain-C fp64 restatement
  (``oracle/bp_oracle.c``) of the reference hot path;
* ``load("ref")`` -> ``oracle/_ref/libbpsched_ref.so``: the UNMODIFIED
  reference core compiled from /root/reference (``oracle/Makefile``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline,
--impl reference) may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "orc": os.path.join(HERE, "liboracle.so"),
    "ref": os.path.join(HERE, "_ref", "libbpsched_ref.so"),
}

KINDS = {"lbp": 0, "srbp": 1, "serial_rbp": 1, "rbp": 2, "rs": 3, "rnbp": 4}


class OrcConfig(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("splash_depth", C.c_uint32),
        ("epsilon", C.c_double),
        ("p", C.c_double),
        ("low_p", C.c_double),
        ("high_p", C.c_double),
        ("edge_ratio_threshold", C.c_double),
        ("max_iterations", C.c_uint64),
        ("time_limit", C.c_double),
        ("seed", C.c_uint64),
        ("worker_count", C.c_uint32),
        ("_pad", C.c_uint32),
    ]


class OrcRecord(C.Structure):
    _fields_ = [
        ("iteration", C.c_uint64),
        ("frontier_size", C.c_uint64),
        ("unconverged", C.c_uint32),
        ("_pad", C.c_uint32),
        ("elapsed_seconds", C.c_double),
    ]


class OrcResult(C.Structure):
    _fields_ = [
        ("converged", C.c_int32),
        ("_pad", C.c_int32),
        ("iterations", C.c_uint64),
        ("wall_time", C.c_double),
        ("messages_updated_total", C.c_uint64),
        ("trace_len", C.c_uint64),
    ]


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def make_config(kind="lbp", epsilon=1e-5, p=1.0, splash_depth=2, low_p=0.7, high_p=1.0,
                edge_ratio_threshold=0.9, max_iterations=10000, time_limit=90.0, seed=0,
                worker_count=0) -> OrcConfig:
    """Defaults of bpsched::SchedulerConfig (schedulers.hpp:26-41)."""
    return OrcConfig(KINDS[kind] if isinstance(kind, str) else int(kind), splash_depth, epsilon, p,
                     low_p, high_p, edge_ratio_threshold, max_iterations, time_limit, seed,
                     worker_count, 0)


_P = C.c_void_p
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C")


class Lib:
    def __init__(self, which: str):
        path = PATHS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run __graft_entry__.build())")
        self.which = which
        self.pre = "orc_" if which == "orc" else "ref_"
        self.lib = C.CDLL(path)
        f = self.fn
        f("last_error", C.c_char_p, [])
        f("graph_create", C.c_int, [C.c_uint32, _u32p, _f64p, C.c_uint32, _u32p, _f64p, C.POINTER(_P)])
        f("graph_destroy", None, [_P])
        f("graph_num_vertices", C.c_uint32, [_P])
        f("graph_num_edges", C.c_uint32, [_P])
        f("graph_unary_size", C.c_uint64, [_P])
        f("graph_table_size", C.c_uint64, [_P])
        f("graph_export", None, [_P, _u32p, _f64p, _u32p, _f64p])
        f("graph_incoming", None, [_P, _u64p, _u32p])
        f("generate_ising", C.c_int, [C.c_uint32, C.c_double, C.c_uint64, C.POINTER(_P)])
        f("generate_chain", C.c_int, [C.c_uint32, C.c_double, C.c_uint64, C.POINTER(_P)])
        if which == "orc":
            f("generate_potts", C.c_int, [C.c_uint32, C.c_uint32, C.c_double, C.c_uint64, C.POINTER(_P)])
            f("generate_er", C.c_int, [C.c_uint32, C.c_uint32, C.c_double, C.c_uint64, C.POINTER(_P)])
            f("engine_set_messages", C.c_int, [_P, _f64p])
        if which == "ref":
            f("parse_model", C.c_int, [C.c_char_p, C.c_uint64, C.POINTER(_P)])
            f("serialize_model", C.c_uint64, [_P, C.c_char_p, C.c_uint64])
        f("mt_draws", None, [C.c_uint64, C.c_uint64, _u64p, _f64p])
        f("validate_config", C.c_int, [C.POINTER(OrcConfig)])
        f("select_parallelism", C.c_double, [C.c_uint32, C.c_uint32, C.POINTER(OrcConfig)])
        f("run", C.c_int, [_P, C.POINTER(OrcConfig), C.POINTER(OrcResult), _P, _P, C.c_uint64])
        f("engine_create", C.c_int, [_P, C.POINTER(OrcConfig), C.POINTER(_P)])
        f("engine_destroy", None, [_P])
        f("engine_unconverged", C.c_uint32, [_P])
        f("engine_iteration", C.c_uint64, [_P])
        f("engine_advance", None, [_P])
        f("engine_messages", None, [_P, _f64p])
        f("engine_candidates", None, [_P, _f64p])
        f("engine_residuals", None, [_P, _f64p])
        f("engine_apply_frontier", C.c_int, [_P, _u32p, C.c_uint64])
        f("engine_frontier_lbp", None, [_P, _u32p, C.POINTER(C.c_uint64)])
        f("engine_rbp_frontier", None, [_P, C.c_double, _u32p, C.POINTER(C.c_uint64)])
        f("engine_rnbp_frontier", None, [_P, C.c_double, _u32p, C.POINTER(C.c_uint64)])
        f("engine_rs_frontier", C.c_int, [_P, C.c_double, C.c_uint32, _u32p, _u64p, _u32p, C.POINTER(C.c_uint64)])
        f("engine_apply_splashes", C.c_int, [_P, C.c_uint64, _u32p, _u64p, _u32p])
        f("engine_beliefs", C.c_int, [_P, _f64p])
        f("engine_build_splash", C.c_int, [_P, C.c_uint32, C.c_uint32, _u32p, _u32p, C.POINTER(C.c_uint64)])
        f("engine_update_message", C.c_int, [_P, C.c_uint32, _f64p])
        f("select_top_k", None, [_f64p, C.c_uint64, C.c_uint64, _u32p, C.POINTER(C.c_uint64)])

    def fn(self, name, restype, argtypes):
        h = getattr(self.lib, self.pre + name)
        h.restype = restype
        h.argtypes = argtypes
        setattr(self, name, h)

    def check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.last_error().decode())


_LIBS: dict = {}


def load(which: str = "orc") -> Lib:
    if which not in _LIBS:
        _LIBS[which] = Lib(which)
    return _LIBS[which]


@dataclass
class GraphArrays:
    """build_graph inputs (mrf.hpp:94-96) as flat arrays."""
    cardinalities: np.ndarray
    unary: np.ndarray
    endpoints: np.ndarray  # (E, 2) uint32
    tables: np.ndarray

    @property
    def num_vertices(self):
        return int(self.cardinalities.size)

    @property
    def num_edges(self):
        return int(self.endpoints.shape[0])


class Graph:
    def __init__(self, lib: Lib, handle):
        self.lib = lib
        self.h = handle

    def __del__(self):
        try:
            if self.h:
                self.lib.graph_destroy(self.h)
        except Exception:
            pass

    @classmethod
    def from_arrays(cls, lib: Lib, cards, unary, endpoints, tables) -> "Graph":
        cards = np.ascontiguousarray(cards, np.uint32)
        unary = np.ascontiguousarray(unary, np.float64)
        ep = np.ascontiguousarray(np.asarray(endpoints, np.uint32).reshape(-1))
        tables = np.ascontiguousarray(tables, np.float64)
        if unary.size == 0:
            unary = np.zeros(1)
        if tables.size == 0:
            tables = np.zeros(1)
        if ep.size == 0:
            ep = np.zeros(2, np.uint32)
        h = _P()
        lib.check(lib.graph_create(cards.size, cards, unary, len(np.asarray(endpoints).reshape(-1)) // 2,
                                   ep, tables, C.byref(h)))
        return cls(lib, h)

    @classmethod
    def parse(cls, lib: Lib, text) -> "Graph":
        """the reference's parse_model (model_io.cpp:98-150); ref only"""
        data = text.encode() if isinstance(text, str) else bytes(text)
        h = _P()
        lib.check(lib.parse_model(data, len(data), C.byref(h)))
        return cls(lib, h)

    def serialize(self) -> str:
        """the reference's serialize_model (model_io.cpp:152-181); ref only"""
        n = self.lib.serialize_model(self.h, None, 0)
        buf = C.create_string_buffer(n)
        self.lib.serialize_model(self.h, buf, n)
        return buf.raw[:n].decode()

    @classmethod
    def ising(cls, lib: Lib, n, c, seed) -> "Graph":
        h = _P()
        lib.check(lib.generate_ising(n, c, seed, C.byref(h)))
        return cls(lib, h)

    @classmethod
    def chain(cls, lib: Lib, n, c, seed) -> "Graph":
        h = _P()
        lib.check(lib.generate_chain(n, c, seed, C.byref(h)))
        return cls(lib, h)

    @classmethod
    def potts(cls, lib: Lib, n, q, c, seed) -> "Graph":
        h = _P()
        lib.check(lib.generate_potts(n, q, c, seed, C.byref(h)))
        return cls(lib, h)

    @classmethod
    def er(cls, lib: Lib, n, m, c, seed) -> "Graph":
        h = _P()
        lib.check(lib.generate_er(n, m, c, seed, C.byref(h)))
        return cls(lib, h)

    @property
    def V(self):
        return int(self.lib.graph_num_vertices(self.h))

    @property
    def E(self):
        return int(self.lib.graph_num_edges(self.h))

    def arrays(self) -> GraphArrays:
        V, E = self.V, self.E
        cards = np.zeros(max(V, 1), np.uint32)
        un = np.zeros(max(int(self.lib.graph_unary_size(self.h)), 1))
        ep = np.zeros(max(2 * E, 2), np.uint32)
        tb = np.zeros(max(int(self.lib.graph_table_size(self.h)), 1))
        self.lib.graph_export(self.h, cards, un, ep, tb)
        return GraphArrays(cards[:V], un[: int(self.lib.graph_unary_size(self.h))],
                           ep[: 2 * E].reshape(E, 2), tb[: int(self.lib.graph_table_size(self.h))])

    def incoming(self):
        off = np.zeros(self.V + 1, np.uint64)
        adj = np.zeros(max(2 * self.E, 1), np.uint32)
        self.lib.graph_incoming(self.h, off, adj)
        return off, adj[: 2 * self.E]

    def message_offsets(self):
        a = self.arrays()
        tgt = np.empty(2 * self.E, np.int64)
        tgt[0::2] = a.endpoints[:, 1]
        tgt[1::2] = a.endpoints[:, 0]
        lens = a.cardinalities[tgt].astype(np.int64)
        return np.concatenate([[0], np.cumsum(lens)])


@dataclass
class RunOut:
    converged: bool
    iterations: int
    wall_time: float
    messages_updated_total: int
    beliefs: np.ndarray
    trace: np.ndarray = field(repr=False)  # (n, 3): iteration, frontier_size, unconverged
    elapsed: np.ndarray = field(repr=False)

    def signature(self):
        """trace_signature (tests/support/test_helpers.hpp:158-166)."""
        s = ("C" if self.converged else "N") + f":{self.iterations}:{self.messages_updated_total}"
        for it, fs, un in self.trace:
            s += f";{it},{fs},{un}"
        return s


def run(g: Graph, cfg: OrcConfig, trace_cap=None) -> RunOut:
    lib = g.lib
    nb = max(int(lib.graph_unary_size(g.h)), 1)
    beliefs = np.zeros(nb)
    if trace_cap is None:
        trace_cap = int(min(cfg.max_iterations, 200000)) + 1
    trace = (OrcRecord * max(trace_cap, 1))()
    res = OrcResult()
    lib.check(lib.run(g.h, C.byref(cfg), C.byref(res), beliefs.ctypes.data_as(_P),
                      C.cast(trace, _P), trace_cap))
    n = min(int(res.trace_len), trace_cap)
    tr = np.array([(trace[k].iteration, trace[k].frontier_size, trace[k].unconverged) for k in range(n)],
                  dtype=np.int64).reshape(n, 3)
    el = np.array([trace[k].elapsed_seconds for k in range(n)])
    return RunOut(bool(res.converged), int(res.iterations), float(res.wall_time),
                  int(res.messages_updated_total), beliefs[: int(lib.graph_unary_size(g.h))], tr, el)


class Engine:
    """Lockstep handle on EngineState (schedulers.hpp:61-90)."""

    def __init__(self, g: Graph, cfg: OrcConfig):
        self.g = g
        self.lib = g.lib
        self.cfg = cfg
        h = _P()
        self.lib.check(self.lib.engine_create(g.h, C.byref(cfg), C.byref(h)))
        self.h = h
        self.D = 2 * g.E
        self.moff = g.message_offsets()

    def __del__(self):
        try:
            if self.h:
                self.lib.engine_destroy(self.h)
        except Exception:
            pass

    @property
    def unconverged(self):
        return int(self.lib.engine_unconverged(self.h))

    @property
    def iteration(self):
        return int(self.lib.engine_iteration(self.h))

    def advance(self):
        self.lib.engine_advance(self.h)

    def messages(self):
        out = np.zeros(max(int(self.moff[-1]), 1))
        self.lib.engine_messages(self.h, out)
        return out[: int(self.moff[-1])]

    def candidates(self):
        out = np.zeros(max(int(self.moff[-1]), 1))
        self.lib.engine_candidates(self.h, out)
        return out[: int(self.moff[-1])]

    def residuals(self):
        out = np.zeros(max(self.D, 1))
        self.lib.engine_residuals(self.h, out)
        return out[: self.D]

    def apply_frontier(self, frontier):
        f = np.ascontiguousarray(frontier, np.uint32)
        if f.size == 0:
            f = np.zeros(1, np.uint32)
            self.lib.check(self.lib.engine_apply_frontier(self.h, f, 0))
        else:
            self.lib.check(self.lib.engine_apply_frontier(self.h, f, f.size))

    def _frontier(self, name, *args):
        out = np.zeros(max(self.D, 1), np.uint32)
        n = C.c_uint64()
        getattr(self.lib, name)(self.h, *args, out, C.byref(n))
        return out[: n.value].copy()

    def frontier_lbp(self):
        return self._frontier("engine_frontier_lbp")

    def rbp_frontier(self, p):
        return self._frontier("engine_rbp_frontier", p)

    def rnbp_frontier(self, p):
        return self._frontier("engine_rnbp_frontier", p)

    def rs_frontier(self, p, h):
        V = self.g.V
        roots = np.zeros(max(V, 1), np.uint32)
        eoff = np.zeros(V + 1, np.uint64)
        edges = np.zeros(max(self.D, 1), np.uint32)
        n = C.c_uint64()
        self.lib.check(self.lib.engine_rs_frontier(self.h, p, h, roots, eoff, edges, C.byref(n)))
        k = n.value
        return roots[:k].copy(), eoff[: k + 1].copy(), edges[: int(eoff[k])].copy()

    def apply_splashes(self, roots, eoff, edges):
        roots = np.ascontiguousarray(roots, np.uint32)
        eoff = np.ascontiguousarray(eoff, np.uint64)
        edges = np.ascontiguousarray(edges, np.uint32)
        self.lib.check(self.lib.engine_apply_splashes(
            self.h, roots.size, roots if roots.size else np.zeros(1, np.uint32), eoff,
            edges if edges.size else np.zeros(1, np.uint32)))

    def build_splash(self, root, h, claimed):
        """build_splash with an explicit root; `claimed` (uint32[V]) is updated in place."""
        edges = np.zeros(max(self.D, 1), np.uint32)
        n = C.c_uint64()
        self.lib.check(self.lib.engine_build_splash(self.h, root, h, claimed, edges, C.byref(n)))
        return edges[: n.value].copy()

    def beliefs(self):
        n = int(self.lib.graph_unary_size(self.g.h))
        out = np.zeros(max(n, 1))
        self.lib.check(self.lib.engine_beliefs(self.h, out))
        return out[:n]

    def set_messages(self, msgs):
        """Load a message state (C restatement only): candidates, residuals and
        the unconverged count are recomputed from it in fp64."""
        self.lib.check(self.lib.engine_set_messages(self.h, np.ascontiguousarray(msgs, np.float64)))

    def update_message(self, d):
        out = np.zeros(max(int(self.moff[d + 1] - self.moff[d]), 1))
        self.lib.check(self.lib.engine_update_message(self.h, d, out))
        return out


def select_top_k(lib: Lib, residuals, k):
    r = np.ascontiguousarray(residuals, np.float64)
    out = np.zeros(max(r.size, 1), np.uint32)
    n = C.c_uint64()
    lib.select_top_k(r if r.size else np.zeros(1), r.size, k, out, C.byref(n))
    return out[: n.value].copy()


def select_parallelism(lib: Lib, prev, now, cfg):
    return lib.select_parallelism(prev, now, C.byref(cfg))


def mt_draws(lib: Lib, seed, count):
    raw = np.zeros(max(count, 1), np.uint64)
    unit = np.zeros(max(count, 1))
    lib.mt_draws(seed, count, raw, unit)
    return raw[:count], unit[:count]
