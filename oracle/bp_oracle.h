/*
 * bp_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C, fp64) of the reference bpsched hot path, used as
 * the parity checker for the CUDA engine.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product library (paper_1909_11469_b200/) never links or calls it.
 *
 * Every function follows the reference's arithmetic order so that results are
 * bitwise identical to the reference compiled with the same flags
 * (-O2 -ffp-contract=off); tests/test_oracle_vs_ref.py pins that against
 * oracle/_ref (the reference itself, compiled from /root/reference).
 */
#ifndef BP_ORACLE_H
#define BP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_INVALID_ARGUMENT = 1, ORC_MODEL = 2, ORC_NUMERIC = 3, ORC_NOMEM = 6 };
enum { ORC_LBP = 0, ORC_SRBP = 1, ORC_RBP = 2, ORC_RS = 3, ORC_RNBP = 4 };

/* Mirrors bpsched::SchedulerConfig (schedulers.hpp:26-41). */
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
} orc_config;

/* Mirrors bpsched::IterationRecord (schedulers.hpp:43-48). */
typedef struct {
  uint64_t iteration;
  uint64_t frontier_size;
  uint32_t unconverged;
  uint32_t _pad;
  double elapsed_seconds;
} orc_record;

/* Mirrors the scalar part of bpsched::RunResult (schedulers.hpp:50-57). */
typedef struct {
  int32_t converged;
  int32_t _pad;
  uint64_t iterations;
  double wall_time;
  uint64_t messages_updated_total;
  uint64_t trace_len;
} orc_result;

typedef struct orc_graph orc_graph;
typedef struct orc_engine orc_engine;

const char* orc_last_error(void);

/* build_graph (mrf.cpp:25-106).  unary: concatenated per-vertex tables;
 * endpoints: (i,j) pairs; tables: concatenated row-major |A_i|x|A_j|. */
int orc_graph_create(uint32_t num_vertices, const uint32_t* cardinalities, const double* unary,
                     uint32_t num_edges, const uint32_t* endpoints, const double* tables,
                     orc_graph** out);
void orc_graph_destroy(orc_graph* g);
uint32_t orc_graph_num_vertices(const orc_graph* g);
uint32_t orc_graph_num_edges(const orc_graph* g);
uint64_t orc_graph_unary_size(const orc_graph* g);
uint64_t orc_graph_table_size(const orc_graph* g);
/* Copies the graph back out in orc_graph_create's layout (any pointer may be NULL). */
void orc_graph_export(const orc_graph* g, uint32_t* cardinalities, double* unary,
                      uint32_t* endpoints, double* tables);
/* CSR of incoming directed edges (mrf.cpp:93-104): offsets[V+1], adjacency[2E]. */
void orc_graph_incoming(const orc_graph* g, uint64_t* offsets, uint32_t* adjacency);

/* generators.cpp:24-71 (bit-identical mt19937_64 streams) + the new Potts/ER
 * instance definitions. */
int orc_generate_ising(uint32_t n, double c, uint64_t seed, orc_graph** out);
int orc_generate_chain(uint32_t length, double c, uint64_t seed, orc_graph** out);
int orc_generate_potts(uint32_t n, uint32_t q, double c, uint64_t seed, orc_graph** out);
int orc_generate_er(uint32_t n, uint32_t m, double c, uint64_t seed, orc_graph** out);

/* mt19937_64 + uniform_unit (rng.hpp:11-13), exposed for tests. */
void orc_mt_draws(uint64_t seed, uint64_t count, uint64_t* out_raw, double* out_unit);

int orc_validate_config(const orc_config* cfg);

/* run (schedulers.cpp:293-353) and run_serial_rbp (serial_rbp.cpp:30-82).
 * beliefs: sum(card) doubles or NULL; trace: trace_cap records or NULL. */
int orc_run(const orc_graph* g, const orc_config* cfg, orc_result* result, double* beliefs,
            orc_record* trace, uint64_t trace_cap);

/* Lockstep access to EngineState (schedulers.hpp:61-90) and its phases. */
int orc_engine_create(const orc_graph* g, const orc_config* cfg, orc_engine** out);
void orc_engine_destroy(orc_engine* e);
uint32_t orc_engine_unconverged(const orc_engine* e);
uint64_t orc_engine_iteration(const orc_engine* e);
void orc_engine_advance(orc_engine* e);
/* Live messages / candidates, linear probabilities, concatenated in directed-edge order. */
void orc_engine_messages(const orc_engine* e, double* out);
void orc_engine_candidates(const orc_engine* e, double* out);
void orc_engine_residuals(const orc_engine* e, double* out);
int orc_engine_apply_frontier(orc_engine* e, const uint32_t* frontier, uint64_t n);
/* Frontier builders; out must hold 2E ids; *n receives the size. */
void orc_engine_frontier_lbp(const orc_engine* e, uint32_t* out, uint64_t* n);
void orc_engine_rbp_frontier(const orc_engine* e, double p, uint32_t* out, uint64_t* n);
void orc_engine_rnbp_frontier(orc_engine* e, double p, uint32_t* out, uint64_t* n);
double orc_select_parallelism(uint32_t prev, uint32_t now, const orc_config* cfg);
/* Splashes: roots[k], edge_offsets[k+1], edges[...]; capacity: roots V, edges 2E. */
int orc_engine_rs_frontier(orc_engine* e, double p, uint32_t h, uint32_t* roots,
                           uint64_t* edge_offsets, uint32_t* edges, uint64_t* num_splashes);
int orc_engine_apply_splashes(orc_engine* e, uint64_t num_splashes, const uint32_t* roots,
                              const uint64_t* edge_offsets, const uint32_t* edges);
int orc_engine_beliefs(const orc_engine* e, double* out);
/* build_splash (schedulers.cpp:136-167) with an explicit root; claimed[V]
 * (UINT32_MAX = unclaimed) is updated; edges capacity 2E. Returns
 * ORC_INVALID_ARGUMENT when the root is already claimed. */
int orc_engine_build_splash(const orc_engine* e, uint32_t root, uint32_t h, uint32_t* claimed,
                            uint32_t* edges, uint64_t* n);
/* One-off update of message d against the live store (messages.cpp:67-73). */
int orc_engine_update_message(const orc_engine* e, uint32_t d, double* out);
/* test aid: load a message state, rebuild candidates / residuals / count (fp64) */
int orc_engine_set_messages(orc_engine* e, const double* msgs);
/* select_top_k (schedulers.cpp:105-116) over an arbitrary residual array. */
void orc_select_top_k(const double* residuals, uint64_t m, uint64_t k, uint32_t* out, uint64_t* n);

#ifdef __cplusplus
}
#endif
#endif
