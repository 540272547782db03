/*
 * bp_cuda.h -- C ABI of the B200 belief-propagation scheduling engine
 * (libbp_b200.so, built from paper_1909_11469_b200/csrc).
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/core, "bpsched"): a PairwiseMRF (mrf.hpp:31-87) plus a
 * SchedulerConfig (schedulers.hpp:26-41) go in, a RunResult
 * (schedulers.hpp:43-57) comes out.  Plain pointers and sizes only; no C++ or
 * torch types cross it.  Each entry point names the reference interface it
 * replaces.  Error convention (schedulers.cpp:78-90, errors.hpp:10-38): every
 * function returns a bp_status; the message of the last failure on the calling
 * thread is available from bp_last_error().  Iteration / time caps are NOT
 * errors (schedulers.cpp:307-309): they yield converged == 0.
 *
 * Threading (mrf.hpp:24-25, schedulers.hpp:59-60): a bp_graph is immutable and
 * may be shared by concurrent runs on its device; a run is synchronous on the
 * calling thread and owns its engine; a bp_engine is not re-entrant.
 */
#ifndef BP_CUDA_H
#define BP_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BP_CUDA_ABI_VERSION 1

#if defined(__GNUC__)
#define BP_API __attribute__((visibility("default")))
#else
#define BP_API
#endif

typedef enum {
  BP_OK = 0,
  BP_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (SchedulerConfig::validate, schedulers.cpp:78-90) */
  BP_ERR_MODEL = 2,            /* bpsched::model_error (errors.hpp:17)   */
  BP_ERR_NUMERIC = 3,          /* bpsched::numeric_error (errors.hpp:23) */
  BP_ERR_CUDA = 4,
  BP_ERR_NCCL = 5,
  BP_ERR_OOM = 6,
  BP_ERR_UNSUPPORTED = 7,
  BP_ERR_PARSE = 8             /* bpsched::parse_error (errors.hpp:29-38): message "line N: ..." */
} bp_status;

/* bpsched::SchedulerKind (schedulers.hpp:21-24), same numbering. */
typedef enum { BP_LBP = 0, BP_SERIAL_RBP = 1, BP_RBP = 2, BP_RS = 3, BP_RNBP = 4 } bp_scheduler_kind;

/* Inputs of bpsched::build_graph (mrf.hpp:94-96), flattened:
 *   unary_values    = concat over v of unary_tables[v]          (sum card)
 *   edge_endpoints  = (i, j) per edge, i < j, edge-id order      (2 E)
 *   pairwise_values = concat over e of the row-major |A_i|x|A_j| table.
 * Arrays are borrowed for the duration of the call only. */
typedef struct {
  uint32_t num_vertices;
  uint32_t num_edges;
  const uint32_t* cardinalities;
  const double* unary_values;
  const uint32_t* edge_endpoints;
  const double* pairwise_values;
} bp_graph_desc;

typedef struct {
  int32_t device;   /* CUDA ordinal, -1 = current */
  uint32_t flags;   /* BP_GRAPH_* */
} bp_device_opts;

#define BP_GRAPH_TRUSTED 1u /* skip the O(E log E) duplicate-edge scan (generated inputs) */

/* bpsched::SchedulerConfig (schedulers.hpp:26-41); worker_count is accepted
 * and ignored (the CUDA grid replaces ThreadPool, thread_pool.hpp:17-45). */
typedef struct {
  int32_t kind;
  uint32_t splash_depth;
  double epsilon;
  double p;
  double low_p;
  double high_p;
  double edge_ratio_threshold;
  uint64_t max_iterations;
  double time_limit;
  uint64_t seed;
  uint32_t worker_count;
  uint32_t _pad;
} bp_sched_config;

/* bpsched::IterationRecord (schedulers.hpp:43-48). */
typedef struct {
  uint64_t iteration;
  uint64_t frontier_size;
  uint32_t unconverged;
  uint32_t _pad;
  double elapsed_seconds;
} bp_iter_record;

/* bpsched::RunResult scalars (schedulers.hpp:50-57) + device statistics. */
typedef struct {
  int32_t converged;
  int32_t stopped;                 /* the run loop has ended (converged or a cap); bp_band_status */
  uint64_t iterations;
  double wall_time;                /* host steady clock, same span as schedulers.cpp:297-350 */
  uint64_t messages_updated_total; /* sum of frontier sizes (schedulers.cpp:343)            */
  uint64_t trace_len;              /* records produced (may exceed trace_cap)               */
  double device_ms;                /* CUDA-event time of the same span on the run's stream  */
  uint64_t message_evaluations;    /* candidate / message recomputations on the device     */
  uint64_t gpu_launches;           /* kernels launched by this run (incl. early-exit ones)  */
  uint64_t vertex_visits;          /* vertices processed by update kernels                  */
  uint64_t splashes;               /* residual splash: splashes applied (all iterations)    */
  uint64_t splash_rounds;          /* residual splash: parallel claiming rounds             */
  uint64_t persist_iterations;     /* RnBP: iterations run inside the persistent tail kernel */
  uint64_t fused_iterations;       /* RnBP: dense iterations run as fused sweeps (k_rnbp_fused) */
} bp_run_result;

typedef struct {
  uint32_t num_vertices;
  uint32_t num_edges;
  uint32_t max_cardinality;
  uint32_t state_stride;  /* floats per message on device (1 = binary log-odds) */
  uint64_t device_bytes;  /* graph bytes resident in HBM */
  int32_t device;
  uint32_t layout;        /* 0 = binary log-odds, 1 = generic log-domain */
  uint64_t message_values;/* sum over directed edges d of card(target(d)): MessageStore size (messages.cpp:23-39) */
} bp_graph_info;

/* Per-kernel-class device time, filled when BP_RUN_KERNEL_TIMING is set. */
#define BP_KERNEL_CLASSES 9
typedef struct {
  /* 0 sweep/refresh, 1 select, 2 radix/top-k, 3 splash, 4 init, 5 beliefs, 6 other,
   * 7 persistent RnBP list-mode tail, 8 fused dense RnBP sweep */
  double ms[BP_KERNEL_CLASSES];
  uint64_t launches[BP_KERNEL_CLASSES];
  uint64_t bytes[BP_KERNEL_CLASSES]; /* algorithmic bytes moved by the timed launches */
} bp_kernel_stats;

typedef struct {
  uint32_t flags;        /* BP_RUN_* */
  uint32_t batch;        /* iterations per device batch (0 = adaptive) */
  bp_kernel_stats* stats;/* optional */
  double* beliefs_device;/* optional: write beliefs (fp64) to this DEVICE pointer instead */
  double* messages_host; /* optional: the live messages at the end of the run as fp64 probabilities,
                            message_values doubles in directed-edge order (MessageStore::view,
                            messages.hpp:24-26; EngineState::messages(), schedulers.hpp:71) */
} bp_run_opts;

#define BP_RUN_KERNEL_TIMING 1u /* CUDA events around every kernel (adds overhead) */
#define BP_RUN_NO_GRAPHS 2u     /* launch kernels directly instead of CUDA-graph batches */
#define BP_RUN_NO_BELIEFS 4u    /* skip beliefs */
#define BP_RUN_NO_PERSIST 8u    /* RnBP: keep the per-kernel graph loop in candidate-list mode */
#define BP_RUN_LBP_TMA 16u      /* LBP: force the TMA-staged lattice sweep (binary Ising lattices, >= 2 rows) */
#define BP_RUN_LBP_TILES 32u    /* LBP: force the register-tiled lattice sweep (default below 2^21 vertices) */
#define BP_RUN_LBP_VERTEX 64u   /* LBP: force the vertex-centric sweep (q-state lattices: instead of lanes over states) */
#define BP_RUN_NO_FUSED 128u    /* RnBP: run the dense iterations as select + refresh launches, not fused sweeps */
#define BP_RUN_FUSED_TMA 256u   /* RnBP: the SMEM-staged fused sweep instead of the register one (slower: DESIGN.md 5) */
#define BP_RUN_FUSED_REGS 512u  /* RnBP: the register fused sweep (the default) */

/* LBP sweep kernels (bp_engine_lbp_sweep's *kernel_out) */
#define BP_LBP_KERNEL_VERTEX 0u /* k_vertex_update: vertex-centric (CSR / generic q-state / Potts lattice) */
#define BP_LBP_KERNEL_TILES 1u  /* k_vertex_update lattice tiles (binary Ising lattice) */
#define BP_LBP_KERNEL_TMA 2u    /* k_lbp_lattice: TMA-staged rows (binary Ising lattice) */
#define BP_LBP_KERNEL_QLANES 3u /* k_lattice_qsweep: q-state lattice, lanes over states (q <= 8, uniform q) */

BP_API const char* bp_last_error(void);
BP_API int bp_abi_version(void);

/* build_graph (mrf.cpp:25-106): validates exactly like the reference (model
 * errors for zero cardinality, table-size mismatch, non-positive / non-finite
 * potentials, self loops, i >= j, duplicates) and uploads to HBM. */
BP_API int bp_graph_create(const bp_graph_desc* desc, const bp_device_opts* opts, struct bp_graph** out);

/* generate_ising / generate_chain (generators.cpp:24-71), bit-identical
 * mt19937_64 streams, built straight into the device layout (no PairwiseMRF
 * on the host: 16384^2 fits).  Potts / Erdos-Renyi: DESIGN.md section 3. */
BP_API int bp_graph_generate_ising(uint32_t n, double c, uint64_t seed, const bp_device_opts* opts,
                            struct bp_graph** out);
BP_API int bp_graph_generate_chain(uint32_t length, double c, uint64_t seed, const bp_device_opts* opts,
                            struct bp_graph** out);
BP_API int bp_graph_generate_potts(uint32_t n, uint32_t q, double c, uint64_t seed,
                            const bp_device_opts* opts, struct bp_graph** out);
BP_API int bp_graph_generate_er(uint32_t n, uint32_t m, double c, uint64_t seed,
                         const bp_device_opts* opts, struct bp_graph** out);

/* Host-side generate_ising in build_graph's input layout (no device work):
 * cards[n*n], unary[2 n*n], endpoints[2E], tables[4E] with E = 2 n (n - 1). */
BP_API int bp_generate_ising_arrays(uint32_t n, double c, uint64_t seed, uint32_t* cardinalities,
                                    double* unary_values, uint32_t* edge_endpoints,
                                    double* pairwise_values);
/* The Erdos-Renyi G(n, m) instance of bp_graph_generate_er as build_graph
 * input arrays (n cardinalities, 2n unaries, 2m endpoints, 4m tables). */
BP_API int bp_generate_er_arrays(uint32_t n, uint32_t m, double c, uint64_t seed, uint32_t* cardinalities,
                                 double* unary, uint32_t* endpoints, double* tables);

/* The reference's text model format (.pgm; parse_model / serialize_model,
 * model_io.cpp:98-181): bulk ingest on the host pool into build_graph's input
 * arrays (BP_ERR_PARSE with the reference's first parse_error, "line N: ...").
 * bp_pgm_*: host only (the arrays); bp_graph_create_pgm: parse + bp_graph_create. */
typedef struct bp_pgm bp_pgm;
BP_API int bp_pgm_parse(const char* text, uint64_t len, bp_pgm** out);
BP_API int bp_pgm_info(const bp_pgm* m, uint32_t* num_vertices, uint32_t* num_edges, uint64_t* unary_len,
                       uint64_t* table_len);
BP_API int bp_pgm_arrays(const bp_pgm* m, uint32_t* cardinalities, double* unary_values, uint32_t* edge_endpoints,
                         double* pairwise_values);
BP_API void bp_pgm_destroy(bp_pgm* m);
BP_API int bp_graph_create_pgm(const char* text, uint64_t len, const bp_device_opts* opts, struct bp_graph** out);

BP_API void bp_graph_destroy(struct bp_graph* g);
BP_API int bp_graph_info_get(const struct bp_graph* g, bp_graph_info* info);

/* bpsched::run (schedulers.hpp:156, schedulers.cpp:293-353).  beliefs_out:
 * sum(card) doubles in vertex order (BeliefTable, messages.hpp:83-107) or NULL;
 * trace_out: trace_cap records or NULL.  kind == BP_SERIAL_RBP returns
 * BP_ERR_UNSUPPORTED: serial RBP is strictly sequential and is
 * not offloaded; the C++ facade routes it to the reference's run_serial_rbp. */
BP_API int bp_run(const struct bp_graph* g, const bp_sched_config* cfg, bp_run_result* result,
           double* beliefs_out, bp_iter_record* trace_out, uint64_t trace_cap);
BP_API int bp_run_ex(const struct bp_graph* g, const bp_sched_config* cfg, const bp_run_opts* opts,
              bp_run_result* result, double* beliefs_out, bp_iter_record* trace_out,
              uint64_t trace_cap);

/* SchedulerConfig::validate (schedulers.cpp:78-90) and select_parallelism
 * (schedulers.cpp:218-224), exported for parity tests. */
BP_API int bp_validate_config(const bp_sched_config* cfg);
BP_API double bp_select_parallelism(uint32_t prev_unconverged, uint32_t new_unconverged,
                             const bp_sched_config* cfg);

/* ---- Lockstep engine: EngineState + per-phase API (schedulers.hpp:61-151) ---- */
BP_API int bp_engine_create(const struct bp_graph* g, const bp_sched_config* cfg, struct bp_engine** out);
BP_API void bp_engine_destroy(struct bp_engine* e);
BP_API int bp_engine_unconverged(const struct bp_engine* e, uint32_t* out);
/* Live messages / candidates as fp64 probabilities, concatenated per directed
 * edge (MessageStore::view, messages.hpp:24-26); residuals fp64 [2E]. */
BP_API int bp_engine_messages(const struct bp_engine* e, double* out);
BP_API int bp_engine_candidates(const struct bp_engine* e, double* out);
BP_API int bp_engine_residuals(const struct bp_engine* e, double* out);
BP_API int bp_engine_beliefs(const struct bp_engine* e, double* out);
/* apply_frontier (schedulers.cpp:226-251): Jacobi commit + touched refresh. */
BP_API int bp_engine_apply_frontier(struct bp_engine* e, const uint32_t* frontier, uint64_t n);
/* apply_splash_frontier (schedulers.cpp:253-291). */
BP_API int bp_engine_apply_splashes(struct bp_engine* e, uint64_t num_splashes, const uint32_t* roots,
                             const uint64_t* edge_offsets, const uint32_t* edges);
/* Device frontier builders; out: capacity 2E ids, ascending id order.
 * rnbp: Philox4x32-10 keyed (seed, iteration, attempt, edge id). */
BP_API int bp_engine_rnbp_frontier(struct bp_engine* e, double p, uint32_t* out, uint64_t* n);
BP_API int bp_engine_rbp_frontier(struct bp_engine* e, double p, uint32_t* out, uint64_t* n);
BP_API int bp_engine_rs_frontier(struct bp_engine* e, double p, uint32_t h, uint32_t* roots,
                          uint64_t* edge_offsets, uint32_t* edges, uint64_t* num_splashes);
/* One full iteration of the configured scheduler (frontier + apply), exactly
 * as one pass of the run loop; *frontier_size receives |F|. */
BP_API int bp_engine_step(struct bp_engine* e, uint64_t* frontier_size);
/* One fused LBP sweep, the kernel bp_run executes per LBP iteration (flags:
 * BP_RUN_LBP_TMA / BP_RUN_LBP_TILES force a lattice kernel).  Sweep t reads
 * m_t and writes m_{t+1} = f(m_t); afterwards bp_engine_messages = m_t,
 * bp_engine_candidates = m_{t+1}, bp_engine_unconverged = #{r(m_t) >= eps},
 * bp_engine_iteration = t: the reference's EngineState after t
 * apply_frontier(frontier_lbp()) calls (schedulers.cpp:99-103, 226-251).
 * The first call re-initialises the messages (init_messages, messages.cpp:23-39).
 * kernel_out (optional): BP_LBP_KERNEL_* that ran.  Residuals are not stored. */
BP_API int bp_engine_lbp_sweep(struct bp_engine* e, uint32_t flags, uint32_t* kernel_out);
BP_API int bp_engine_iteration(const struct bp_engine* e, uint64_t* out);
/* EngineState::advance_iteration (schedulers.hpp:75): the next rnbp_frontier
 * draws with the next iteration's Philox keys */
BP_API int bp_engine_advance_iteration(struct bp_engine* e);

/* ---- Row-band partition of a lattice across GPUs ----------
 * Rank `part` of `nparts` owns rows [row0, row1) of generate_ising(n, c, seed)
 * (generators.cpp:24-50); its band adds one ghost row per neighbouring band.
 * Per LBP iteration the caller runs, in order on bp_band_stream():
 *   bp_band_lbp_sweep   sweep of the band, boundary messages -> send_up /
 *                       send_down, local unconverged count + time vote -> count[0..1]
 *   (collectives)       send_up -> rank-1's recv_down, send_down -> rank+1's
 *                       recv_up, all-reduce(sum) of count[0..1]
 *   bp_band_lbp_finish  ghost messages <- recv_*, run() loop control on the
 *                       GLOBAL count (every rank takes the same stop decision)
 * Owned messages are bitwise identical to the unpartitioned run. */
typedef struct {
  uint32_t part, nparts;
  uint32_t row0, row1;          /* owned global rows [row0, row1) */
  uint32_t ghost_up, ghost_down;
  uint32_t local_rows, cols;    /* band lattice: local_rows x cols */
  uint64_t owned_directed;      /* directed edges whose source row is owned */
} bp_band_info;

typedef struct {                /* DEVICE pointers, owned by the caller */
  float* send_up;               /* cols floats */
  float* send_down;             /* cols floats */
  const float* recv_up;         /* cols floats */
  const float* recv_down;       /* cols floats */
  unsigned long long* count;    /* 2 values, all-reduced (sum) in place between sweep and finish */
} bp_halo_buffers;

BP_API int bp_graph_generate_ising_band(uint32_t n, double c, uint64_t seed, uint32_t part, uint32_t nparts,
                                        const bp_device_opts* opts, struct bp_graph** out, bp_band_info* info);
BP_API int bp_band_engine_create(const struct bp_graph* g, const bp_sched_config* cfg, const bp_band_info* info,
                                 const bp_halo_buffers* bufs, struct bp_engine** out);
BP_API int bp_band_stream(const struct bp_engine* e, uint64_t* stream); /* cudaStream_t of the band */
BP_API int bp_band_lbp_sweep(struct bp_engine* e);
BP_API int bp_band_lbp_finish(struct bp_engine* e);
BP_API int bp_band_status(struct bp_engine* e, bp_run_result* result); /* synchronises */

/* RnBP on a band (same row partition; count[] holds 5 values: {delta,
 * frontier, survivors, time vote, initial count}).  Per iteration, on
 * bp_band_stream():
 *   bp_band_rnbp_select(e, 0)  rnbp_frontier attempt 0 over the owned edges
 *                              (Philox keyed by GLOBAL edge ids) + Jacobi
 *                              commit; boundary messages -> send_*
 *   (exchange)                 halos as for LBP
 *   bp_band_rnbp_refresh       ghost messages <- recv_* (a changed one flags
 *                              the owned vertex it flows into), touched
 *                              refresh, sums -> count[0..4]
 *   (all-reduce count)
 *   if the global frontier is 0 and survivors exist (schedulers.cpp:204-214):
 *     select(e, 1) + exchange + refresh + all-reduce; still 0 -> every rank
 *     lists its survivors (bp_band_survivors), the survivor of global rank
 *     min(S-1, floor(u S)) in ascending global id (u = bp_philox_u53(seed,
 *     iteration, 2, 0) * 2^-53) is committed by its owner
 *     (bp_band_rnbp_fallback; the others pass UINT64_MAX) + exchange +
 *     refresh + all-reduce
 *   bp_band_rnbp_finish        loop control on the global sums
 * before the loop: bp_band_rnbp_begin + all-reduce + bp_band_rnbp_finish_init. */
BP_API int bp_band_rnbp_begin(struct bp_engine* e);
BP_API int bp_band_rnbp_finish_init(struct bp_engine* e);
BP_API int bp_band_rnbp_select(struct bp_engine* e, uint32_t attempt);
BP_API int bp_band_rnbp_refresh(struct bp_engine* e);
/* RBP on a band: the band's local top-k (k = max(1, llround(p * owned directed
 * edges)), ties to the lower id) + commit + pack; then refresh / all-reduce /
 * finish exactly as RnBP (no retry).  Per-partition local frontiers (SURVEY
 * 8(e)): differs from the global select_top_k when P > 1, by design. */
BP_API int bp_band_rbp_select(struct bp_engine* e);
/* Residual Splash on a band: local splashes (roots and claims on owned
 * vertices, k = max(1, llround(p * owned vertices))) + commit + pack; then as
 * RnBP.  Per-partition local frontiers, by design. */
BP_API int bp_band_rs_select(struct bp_engine* e);
BP_API int bp_band_rnbp_finish(struct bp_engine* e);
BP_API int bp_band_survivors(struct bp_engine* e, uint64_t* global_ids, uint64_t cap, uint64_t* n);

/* ---- Row-band partition driven from C++ (no Python in the loop) ----------
 * bp_graph_create_band: band `part` of `nparts` of ANY binary Ising lattice
 *   given in build_graph's input layout (generate_ising's edge numbering,
 *   generators.cpp:37-43; any rows x cols; tables {a, d, d, a}); owned rows
 *   [row0, row1) of R rows plus one ghost row per neighbouring band.
 * bp_band_engine_create_owned: a band engine that owns its halo buffers.
 * bp_band_comm_create_nccl: the ranks' NCCL communicator (every rank passes
 *   the same 128-byte id from bp_nccl_unique_id on one rank; libnccl.so.2 is
 *   loaded at first use).  bp_band_comm_create_local: all bands in this
 *   process (host-staged copies; tests on one GPU).
 * bp_band_run: the run() loop (schedulers.cpp:301-347) of LBP / RnBP / RBP /
 *   RS over the bands -- NCCL: nbands == 1, this rank's band; local: the
 *   bands of parts 0 .. P-1 in order.  Halo send/recv and the all-reduce of
 *   the loop counters are enqueued on the band's stream; the loop control
 *   runs on the device from the global counts, so every rank stops at the
 *   same iteration and owned messages equal the unpartitioned run's bit for
 *   bit (LBP, RnBP).  The host polls every 16 iterations; an RnBP iteration
 *   with an empty global attempt-0 frontier parks the bands until the poll
 *   runs the retry / single-survivor fallback (schedulers.cpp:204-214).
 *   result: the global iteration count / convergence; messages_updated_total
 *   counts this band's owned messages (LBP) or the global frontier (others).
 *   Beliefs of the owned rows: bp_engine_beliefs (rows row0 - ghost_up ... in
 *   local numbering). */
typedef struct bp_band_comm bp_band_comm;
BP_API int bp_graph_create_band(const bp_graph_desc* desc, uint32_t part, uint32_t nparts,
                                const bp_device_opts* opts, struct bp_graph** out, bp_band_info* info);
BP_API int bp_band_engine_create_owned(const struct bp_graph* g, const bp_sched_config* cfg,
                                       const bp_band_info* info, struct bp_engine** out);
BP_API int bp_nccl_unique_id(uint8_t* id /* 128 bytes */);
BP_API int bp_band_comm_create_nccl(const uint8_t* id, uint32_t rank, uint32_t nranks, int32_t device,
                                    bp_band_comm** out);
BP_API int bp_band_comm_create_local(bp_band_comm** out);
BP_API void bp_band_comm_destroy(bp_band_comm* c);
BP_API int bp_band_run(struct bp_engine* const* bands, uint32_t nbands, bp_band_comm* comm, bp_run_result* result);
BP_API int bp_band_rnbp_fallback(struct bp_engine* e, uint64_t global_d);

/* ---- Vertex-range partition of ANY binary pairwise MRF (north_star: LBP and
 * RnBP on large grids and random graphs partitioned across GPUs) ------------
 * bp_graph_create_part: part `part` of `nparts` owns global vertices
 *   [v0, v1) = [V part / nparts, V (part + 1) / nparts) and every message whose
 *   source it owns.  Its local graph holds the edges with an owned endpoint
 *   (global order and orientation; build_graph's validation runs on the whole
 *   model, mrf.cpp:28-91) with local vertices = the owned ones in order, then
 *   one ghost per outside neighbour.  Every iteration the messages that cross
 *   the cut move to the part that owns their target (one send / recv run per
 *   peer part, ordered by global directed id on both sides).
 * bp_part_engine_create: its engine with owned halo buffers; drive the parts
 *   with bp_band_run (NCCL: one part per rank; local: parts 0 .. P-1 in this
 *   process).  LBP owned messages and RnBP runs (draws keyed by GLOBAL edge
 *   ids) are identical to the unpartitioned run; beliefs of local vertices
 *   [0, v1 - v0) are the owned ones. */
typedef struct {
  uint32_t part, nparts;
  uint32_t v0, v1;              /* owned global vertices [v0, v1) = local [0, v1 - v0) */
  uint32_t ghost_vertices;      /* local [v1 - v0, v1 - v0 + ghost_vertices) */
  uint32_t local_edges;
  uint32_t peers;               /* parts exchanging cut messages with this one */
  uint32_t _pad;
  uint64_t send_messages, recv_messages;  /* cut messages per iteration (all peers) */
  uint64_t owned_directed;      /* directed edges whose source is owned */
} bp_part_info;
BP_API int bp_graph_create_part(const bp_graph_desc* desc, uint32_t part, uint32_t nparts,
                                const bp_device_opts* opts, struct bp_graph** out, bp_part_info* info);
BP_API int bp_part_engine_create(const struct bp_graph* g, const bp_sched_config* cfg, struct bp_engine** out);
BP_API uint64_t bp_philox_u53(uint64_t seed, uint64_t iteration, uint32_t attempt, uint64_t d);

/* ---- Diagnostics: the DEVICE random stream, for known-answer tests ---------
 * bp_philox4x32_10_device: the device's Philox4x32-10 (Salmon et al., SC'11;
 * Random123 philox4x32_R with R = 10) on n (counter[4], key[2]) pairs.
 * bp_philox_u53_device: the 53-bit RnBP draw of directed edge d[i] in
 * (seed, iteration, attempt), as k_rnbp_select draws it (u = value * 2^-53,
 * the device analogue of uniform_unit, rng.hpp:11-13).  device: -1 = current. */
BP_API int bp_philox4x32_10_device(int32_t device, uint64_t n, const uint32_t* ctr, const uint32_t* key,
                                   uint32_t* out);
BP_API int bp_philox_u53_device(int32_t device, uint64_t seed, uint64_t iteration, uint32_t attempt, uint64_t n,
                                const uint64_t* d, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* BP_CUDA_H */
