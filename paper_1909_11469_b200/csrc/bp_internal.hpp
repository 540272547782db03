// Host-side internals of libbp_b200.so (not part of the ABI).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bp_cuda.h"

namespace bpb {

// Exceptions mirror the reference hierarchy (errors.hpp:10-38); the C ABI
// maps each to its bp_status.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void throw_model(const std::string& m) { throw Error(BP_ERR_MODEL, m); }
[[noreturn]] inline void throw_invalid(const std::string& m) { throw Error(BP_ERR_INVALID_ARGUMENT, m); }

// mt19937_64 with the reference's uniform_unit (rng.hpp:11-13): std::mt19937_64
// has a fully specified sequence, so this is bit-identical across platforms.
class Mt64 {
 public:
  explicit Mt64(uint64_t seed);
  uint64_t next();
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double unit_open() {  // generators.cpp:9-14
    double u = unit();
    while (u == 0.0) u = unit();
    return u;
  }

 private:
  uint64_t mt_[312];
  int idx_;
};

// Host-side instance streams (generators.cpp:24-71 for Ising/chain; the new
// Potts and Erdos-Renyi definitions are in DESIGN.md section 3).
struct BinaryStreams {
  std::vector<float> unary_lo;  // log2(u1) - log2(u0) per vertex (binary layout: base-2 log-odds)
  std::vector<float> coupling;  // J = 2 * lambda * c per edge (log-table differences)
};
BinaryStreams ising_streams(uint32_t n, double c, uint64_t seed);
BinaryStreams ising_band_streams(uint32_t n, double c, uint64_t seed, uint32_t a, uint32_t b);
BinaryStreams chain_streams(uint32_t length, double c, uint64_t seed);

struct PottsStreams {
  std::vector<float> unary_log;  // V * q, log2(u) (device layout: base-2 logs)
  std::vector<float> lambda_c;   // lambda * c per edge
};
PottsStreams potts_streams(uint32_t n, uint32_t q, double c, uint64_t seed);

struct ErInstance {
  std::vector<uint32_t> endpoints;  // 2m, sorted (lo, hi)
  std::vector<float> unary_lo;
  std::vector<float> coupling;
};
ErInstance er_instance(uint32_t n, uint32_t m, double c, uint64_t seed);
// the same instance as build_graph input arrays (unaries, Ising tables {a, d, d, a})
void er_desc_arrays(uint32_t n, uint32_t m, double c, uint64_t seed, std::vector<uint32_t>& cards,
                    std::vector<double>& unary, std::vector<uint32_t>& ep, std::vector<double>& tables);

// The reference's text model (.pgm, model_io.cpp:98-150) as build_graph's
// input arrays (pgm.cpp); throws Error(BP_ERR_PARSE, "line N: ...") as
// parse_model throws parse_error.
struct PgmArrays {
  std::vector<uint32_t> cards, ep;
  std::vector<double> unary, tables;
};
void parse_pgm(const char* text, size_t len, PgmArrays& out);

// Exact double-precision unary / table values of the same streams (for the
// descriptor path and tests).
void ising_desc_arrays(uint32_t rows, uint32_t cols, double c, uint64_t seed,
                       std::vector<uint32_t>& cards, std::vector<double>& unary,
                       std::vector<uint32_t>& ep, std::vector<double>& tables);

}  // namespace bpb
