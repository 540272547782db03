// Bulk ingest of the reference's text model format (`.pgm`, model_io.cpp:98-181)
// straight into build_graph's input arrays: the model
// text is tokenised and converted on the host pool -- line-aligned chunks are
// independent because a comment ends at its newline -- so a million-vertex
// model parses in milliseconds instead of going through the reference's
// sequential parse_model + per-edge std::vector tables.
//
// Fast path: uniform cardinalities (the token layout is then arithmetic:
// header 4, cards V, unaries V q, per edge 2 + q^2).  Anything else -- mixed
// cardinalities, a token count that does not match, any malformed or
// out-of-range token -- runs the sequential restatement of parse_model
// (parse_sequential), which raises the reference's first parse_error with its
// message and line ("line N: ...", errors.hpp:29-38).
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstring>
#include <string>
#include <string_view>
#include <vector>

#include "bp_internal.hpp"
#include "host_pool.hpp"

namespace bpb {

namespace {

inline bool is_sep(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }

[[noreturn]] void throw_parse(const std::string& what, int line) {
  throw Error(BP_ERR_PARSE, "line " + std::to_string(line) + ": " + what);
}

// The reference's Tokenizer (model_io.cpp:14-88), restated.
class SeqTokens {
 public:
  explicit SeqTokens(std::string_view t) : t_(t) {}
  int line() const { return line_; }
  bool at_end() {
    skip();
    return pos_ == t_.size();
  }
  std::string_view next(const char* expectation) {
    skip();
    if (pos_ == t_.size()) throw_parse(std::string("expected ") + expectation + ", got end of input", line_);
    const size_t s = pos_;
    while (pos_ < t_.size() && !is_sep(t_[pos_]) && t_[pos_] != '#') ++pos_;
    return t_.substr(s, pos_ - s);
  }
  uint64_t next_count(const char* expectation) {
    const int at = line_;
    const std::string_view tok = next(expectation);
    uint64_t v = 0;
    const auto [p, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), v);
    if (ec != std::errc{} || p != tok.data() + tok.size())
      throw_parse(std::string("expected ") + expectation + ", got '" + std::string(tok) + "'", at);
    return v;
  }
  double next_real(const char* expectation) {
    const int at = line_;
    const std::string_view tok = next(expectation);
    double v = 0.0;
    const auto [p, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), v);
    if (ec != std::errc{} || p != tok.data() + tok.size())
      throw_parse(std::string("expected ") + expectation + ", got '" + std::string(tok) + "'", at);
    if (!std::isfinite(v)) throw_parse("non-finite number '" + std::string(tok) + "'", at);
    return v;
  }

 private:
  void skip() {
    while (pos_ < t_.size()) {
      const char c = t_[pos_];
      if (c == '\n') {
        ++line_;
        ++pos_;
      } else if (is_sep(c)) {
        ++pos_;
      } else if (c == '#') {
        while (pos_ < t_.size() && t_[pos_] != '\n') ++pos_;
      } else {
        break;
      }
    }
  }
  std::string_view t_;
  size_t pos_ = 0;
  int line_ = 1;
};

// parse_model (model_io.cpp:98-150) up to build_graph, restated: the error
// path of the fast parser, and the path of mixed-cardinality models
void parse_sequential(std::string_view text, PgmArrays& out) {
  SeqTokens tok(text);
  const std::string_view magic = tok.next("'pgm' header");
  if (magic != "pgm") throw_parse("expected 'pgm' header, got '" + std::string(magic) + "'", tok.line());
  const uint64_t V = tok.next_count("vertex count");
  const uint64_t E = tok.next_count("edge count");
  const uint64_t version = tok.next_count("format version");
  if (version != 0) throw_parse("unsupported format version " + std::to_string(version), tok.line());
  if (V > 0xFFFFFFFFull || E > 0xFFFFFFFFull) throw Error(BP_ERR_MODEL, "model too large for 32-bit ids");
  out.cards.assign(V, 0);
  for (uint64_t v = 0; v < V; ++v) {
    const uint64_t c = tok.next_count("cardinality");
    if (c == 0 || c > 0xFFFFFFFFull) throw_parse("cardinality out of range", tok.line());
    out.cards[v] = static_cast<uint32_t>(c);
  }
  out.unary.clear();
  for (uint64_t v = 0; v < V; ++v)
    for (uint32_t x = 0; x < out.cards[v]; ++x) out.unary.push_back(tok.next_real("unary entry"));
  out.ep.assign(2 * E, 0);
  out.tables.clear();
  for (uint64_t e = 0; e < E; ++e) {
    const int at = tok.line();
    const uint64_t i = tok.next_count("edge endpoint");
    const uint64_t j = tok.next_count("edge endpoint");
    if (i >= V || j >= V) throw_parse("edge endpoint out of range", at);
    out.ep[2 * e] = static_cast<uint32_t>(i);
    out.ep[2 * e + 1] = static_cast<uint32_t>(j);
    const size_t n = static_cast<size_t>(out.cards[i]) * out.cards[j];
    for (size_t t = 0; t < n; ++t) out.tables.push_back(tok.next_real("pairwise entry"));
  }
  if (!tok.at_end()) throw_parse("unexpected trailing token '" + std::string(tok.next("")) + "'", tok.line());
}

// tokens of one line-aligned chunk: f(global token index, token)
template <class F>
void walk_tokens(const char* p, size_t a, size_t b, uint64_t k0, F&& f) {
  size_t i = a;
  uint64_t k = k0;
  while (i < b) {
    const char c = p[i];
    if (is_sep(c)) {
      ++i;
    } else if (c == '#') {
      while (i < b && p[i] != '\n') ++i;
    } else {
      const size_t s = i;
      while (i < b && !is_sep(p[i]) && p[i] != '#') ++i;
      if (!f(k++, std::string_view(p + s, i - s))) return;
    }
  }
}

}  // namespace

void parse_pgm(const char* text, size_t len, PgmArrays& out) {
  const std::string_view all(text, len);
  // line-aligned chunks (a comment ends at its newline: chunks are independent)
  const unsigned nch = static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(len >> 20, 4u * HostPool::get().size())));
  std::vector<size_t> start(nch + 1, len);
  start[0] = 0;
  for (unsigned c = 1; c < nch; ++c) {
    size_t s = std::max(start[c - 1], len * c / nch);
    while (s < len && text[s - 1] != '\n') ++s;
    start[c] = s;
  }
  std::vector<uint64_t> ntok(nch + 1, 0);
  HostPool::get().run(nch, [&](unsigned c) {
    uint64_t n = 0;
    walk_tokens(text, start[c], start[c + 1], 0, [&](uint64_t, std::string_view) {
      ++n;
      return true;
    });
    ntok[c + 1] = n;
  });
  for (unsigned c = 0; c < nch; ++c) ntok[c + 1] += ntok[c];
  // header (tokens 0..3) and the cardinalities decide the layout
  uint64_t hdr[3] = {0, 0, 0};
  bool ok = ntok[nch] >= 4;
  if (ok) {
    int got = 0;
    walk_tokens(text, 0, len, 0, [&](uint64_t k, std::string_view t) {
      if (k == 0) {
        ok = t == "pgm";
      } else {
        const auto [p, ec] = std::from_chars(t.data(), t.data() + t.size(), hdr[k - 1]);
        ok = ok && ec == std::errc{} && p == t.data() + t.size();
      }
      return ++got < 4;
    });
  }
  const uint64_t V = hdr[0], E = hdr[1];
  ok = ok && hdr[2] == 0 && V <= 0xFFFFFFFFull && E <= 0xFFFFFFFFull && ntok[nch] >= 4 + V;
  std::atomic<bool> bad{!ok};
  if (ok) {
    out.cards.assign(V, 0);
    HostPool::get().run(nch, [&](unsigned c) {
      if (ntok[c + 1] <= 4 || ntok[c] >= 4 + V) return;
      walk_tokens(text, start[c], start[c + 1], ntok[c], [&](uint64_t k, std::string_view t) {
        if (k >= 4 + V) return false;
        if (k < 4) return true;
        uint64_t v = 0;
        const auto [p, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
        if (ec != std::errc{} || p != t.data() + t.size() || v == 0 || v > 0xFFFFFFFFull) {
          bad = true;
          return false;
        }
        out.cards[k - 4] = static_cast<uint32_t>(v);
        return true;
      });
    });
  }
  const uint32_t q = ok && V ? out.cards[0] : 2u;
  if (!bad && V && std::any_of(out.cards.begin(), out.cards.end(), [&](uint32_t c) { return c != q; })) bad = true;
  const uint64_t base_u = 4 + V, base_e = base_u + V * q, per_e = 2 + static_cast<uint64_t>(q) * q;
  if (!bad && ntok[nch] != base_e + E * per_e) bad = true;  // missing / trailing tokens: the sequential message
  if (!bad) {
    out.unary.assign(V * q, 0.0);
    out.ep.assign(2 * E, 0);
    out.tables.assign(E * q * q, 0.0);
    HostPool::get().run(nch, [&](unsigned c) {
      if (ntok[c + 1] <= base_u) return;
      walk_tokens(text, start[c], start[c + 1], ntok[c], [&](uint64_t k, std::string_view t) {
        if (k < base_u) return true;
        if (k < base_e || (k - base_e) % per_e >= 2) {
          double v = 0.0;
          const auto [p, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
          if (ec != std::errc{} || p != t.data() + t.size() || !std::isfinite(v)) {
            bad = true;
            return false;
          }
          if (k < base_e) {
            out.unary[k - base_u] = v;
          } else {
            const uint64_t e = (k - base_e) / per_e, w = (k - base_e) % per_e;
            out.tables[e * q * q + (w - 2)] = v;
          }
        } else {
          uint64_t v = 0;
          const auto [p, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
          if (ec != std::errc{} || p != t.data() + t.size() || v >= V) {
            bad = true;
            return false;
          }
          const uint64_t e = (k - base_e) / per_e, w = (k - base_e) % per_e;
          out.ep[2 * e + w] = static_cast<uint32_t>(v);
        }
        return true;
      });
    });
  }
  if (bad) parse_sequential(all, out);  // raises the reference's first error (or parses a mixed model)
}

}  // namespace bpb
