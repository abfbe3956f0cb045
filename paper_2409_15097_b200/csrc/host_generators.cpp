// host_generators.cpp — mask families used as fixtures (the reference's generators.hpp).
//
// These build the bit-packed masks the configs are quoted on; they are not on the attention
// path. The spec grammar and every family follow generators.hpp: MEDUSA tree (:22-63), causal /
// all-ones (:65-79), packed sequential (:83-98), packed input-bidirectional (:103-124),
// Longformer windowed / dilated / global (:127-166), random sparse (:171-183), and the spec
// string grammar (:364-438). Random draws use std::mt19937_64 with the reference's
// implementation-independent mapping (rng.hpp:15-17), so seeded masks are bit-identical.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/bbm_capi.h"
#include "bbm_internal.h"

namespace {

using bbm::ArgError;
using bbm::require;

struct Bits {
  uint64_t n, wpr;
  std::vector<uint64_t> w;
  explicit Bits(uint64_t n_) : n(n_), wpr((n_ + 63) / 64), w(n_ * ((n_ + 63) / 64), 0) {}
  void set(uint64_t i, uint64_t j) { w[i * wpr + (j >> 6)] |= 1ull << (j & 63); }
  void set_range(uint64_t i, uint64_t j0, uint64_t j1) {  // [j0, j1)
    for (uint64_t j = j0; j < j1;) {
      if ((j & 63) == 0 && j + 64 <= j1) {
        w[i * wpr + (j >> 6)] = ~0ull;
        j += 64;
      } else {
        set(i, j);
        ++j;
      }
    }
  }
};

double unit(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  size_t start = 0;
  for (;;) {
    const size_t pos = s.find(sep, start);
    if (pos == std::string::npos) {
      out.push_back(s.substr(start));
      return out;
    }
    out.push_back(s.substr(start, pos - start));
    start = pos + 1;
  }
}

uint64_t to_size(const std::string& s) {
  require(!s.empty() && s.find_first_not_of("0123456789") == std::string::npos,
          "bad integer in mask spec: '" + s + "'");
  return std::stoull(s);
}

double to_double(const std::string& s) {
  size_t used = 0;
  double v = 0.0;
  try {
    v = std::stod(s, &used);
  } catch (const std::exception&) {
    throw ArgError("bad number in mask spec: '" + s + "'");
  }
  require(used == s.size(), "bad number in mask spec: '" + s + "'");
  return v;
}

std::vector<std::pair<std::string, std::string>> kv(const std::string& body) {
  std::vector<std::pair<std::string, std::string>> out;
  if (body.empty()) return out;
  for (const auto& item : split(body, ';')) {
    const size_t eq = item.find('=');
    require(eq != std::string::npos, "expected key=value in mask spec: '" + item + "'");
    out.emplace_back(item.substr(0, eq), item.substr(eq + 1));
  }
  return out;
}

Bits medusa(const std::vector<uint64_t>& cand) {
  require(!cand.empty(), "medusa candidate list must be non-empty");
  uint64_t n = 0, level = 1;
  for (uint64_t s : cand) {
    require(s >= 1, "medusa candidate counts must be positive");
    level *= s;
    n += level;
  }
  Bits m(n);
  std::vector<uint64_t> parent(n);
  uint64_t start = 0, size = cand[0];
  for (uint64_t t = 0; t < size; ++t) parent[t] = t;
  for (size_t k = 1; k < cand.size(); ++k) {
    const uint64_t next = start + size;
    for (uint64_t t = 0; t < size * cand[k]; ++t) parent[next + t] = start + t / cand[k];
    start = next;
    size *= cand[k];
  }
  for (uint64_t i = 0; i < n; ++i) {
    m.set(i, i);
    for (uint64_t node = i; parent[node] != node;) {
      node = parent[node];
      m.set(i, node);
    }
  }
  return m;
}

Bits causal(uint64_t n) {
  require(n >= 1, "n must be positive");
  Bits m(n);
  for (uint64_t i = 0; i < n; ++i) m.set_range(i, 0, i + 1);
  return m;
}

Bits all_ones(uint64_t n) {
  require(n >= 1, "n must be positive");
  Bits m(n);
  for (uint64_t i = 0; i < n; ++i) m.set_range(i, 0, n);
  return m;
}

Bits packed_seq(const std::vector<uint64_t>& lens) {
  require(!lens.empty(), "length list must be non-empty");
  uint64_t n = 0;
  for (uint64_t l : lens) {
    require(l >= 1, "segment lengths must be positive");
    n += l;
  }
  Bits m(n);
  uint64_t s = 0;
  for (uint64_t l : lens) {
    for (uint64_t i = s; i < s + l; ++i) m.set_range(i, s, i + 1);
    s += l;
  }
  return m;
}

Bits packed_bidir(const std::vector<std::pair<uint64_t, uint64_t>>& segs) {
  require(!segs.empty(), "segment list must be non-empty");
  uint64_t n = 0;
  for (auto [a, b] : segs) {
    require(a + b >= 1, "segments must be non-empty");
    n += a + b;
  }
  Bits m(n);
  uint64_t s = 0;
  for (auto [in, out] : segs) {
    const uint64_t o = s + in;
    for (uint64_t i = s; i < o; ++i) m.set_range(i, s, o);
    for (uint64_t i = o; i < o + out; ++i) {
      m.set_range(i, s, o);
      m.set_range(i, o, i + 1);
    }
    s += in + out;
  }
  return m;
}

Bits windowed(uint64_t n, uint64_t w, bool causal_only) {
  require(n >= 1, "n must be positive");
  require(w < n, "window must be < n");
  Bits m(n);
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t j0 = i >= w ? i - w : 0;
    const uint64_t j1 = causal_only ? i : std::min(i + w, n - 1);
    m.set_range(i, j0, j1 + 1);
  }
  return m;
}

Bits dilated(uint64_t n, uint64_t w, uint64_t d) {
  require(n >= 1, "n must be positive");
  require(w < n, "window must be < n");
  require(d >= 1, "dilation must be >= 1");
  Bits m(n);
  const uint64_t reach = w * d;
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t step = 0; step <= reach; step += d) {
      if (step <= i) m.set(i, i - step);
      if (i + step < n) m.set(i, i + step);
    }
  return m;
}

Bits global_mask(uint64_t n, uint64_t w, uint64_t g) {
  require(g <= n, "global token count must be <= n");
  Bits m = windowed(n, w, false);
  for (uint64_t t = 0; t < g; ++t) {
    m.set_range(t, 0, n);
    for (uint64_t i = 0; i < n; ++i) m.set(i, t);
  }
  return m;
}

Bits random_sparse(uint64_t n, double p, uint64_t seed, bool diag) {
  require(n >= 1, "n must be positive");
  require(p >= 0.0 && p <= 1.0, "density must be in [0, 1]");
  Bits m(n);
  std::mt19937_64 gen(seed);
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t j = 0; j < n; ++j)
      if (unit(gen) < p) m.set(i, j);
  if (diag)
    for (uint64_t i = 0; i < n; ++i) m.set(i, i);
  return m;
}

Bits parse_and_generate(const std::string& text, uint64_t n_free) {
  std::string name = text, body;
  const size_t open = text.find_first_of("[(");
  if (open != std::string::npos) {
    const char close = text[open] == '[' ? ']' : ')';
    require(text.back() == close, "unbalanced bracket in mask spec: '" + text + "'");
    name = text.substr(0, open);
    body = text.substr(open + 1, text.size() - open - 2);
  }
  if (name == "causal") return causal(n_free);
  if (name == "all-ones") return all_ones(n_free);
  if (name == "medusa") {
    std::vector<uint64_t> c;
    for (const auto& it : split(body, ';')) c.push_back(to_size(it));
    return medusa(c);
  }
  if (name == "packed-seq") {
    std::vector<uint64_t> l;
    for (const auto& it : split(body, ';')) l.push_back(to_size(it));
    return packed_seq(l);
  }
  if (name == "packed-bidir") {
    std::vector<std::pair<uint64_t, uint64_t>> segs;
    for (const auto& it : split(body, ';')) {
      const auto parts = split(it, ':');
      require(parts.size() == 2, "expected in:out segment in mask spec: '" + it + "'");
      segs.emplace_back(to_size(parts[0]), to_size(parts[1]));
    }
    return packed_bidir(segs);
  }
  if (name == "windowed") {
    uint64_t w = 0;
    bool c = false;
    for (const auto& [k, v] : kv(body)) {
      if (k == "w") w = to_size(v);
      else if (k == "causal") c = to_size(v) != 0;
      else throw ArgError("unknown windowed parameter: " + k);
    }
    return windowed(n_free, w, c);
  }
  if (name == "dilated") {
    uint64_t w = 0, d = 1;
    for (const auto& [k, v] : kv(body)) {
      if (k == "w") w = to_size(v);
      else if (k == "d") d = to_size(v);
      else throw ArgError("unknown dilated parameter: " + k);
    }
    return dilated(n_free, w, d);
  }
  if (name == "global") {
    uint64_t w = 0, g = 0;
    for (const auto& [k, v] : kv(body)) {
      if (k == "w") w = to_size(v);
      else if (k == "g") g = to_size(v);
      else throw ArgError("unknown global parameter: " + k);
    }
    return global_mask(n_free, w, g);
  }
  if (name == "random") {
    double p = 0.0;
    uint64_t seed = 0;
    bool diag = true;
    for (const auto& [k, v] : kv(body)) {
      if (k == "p") p = to_double(v);
      else if (k == "seed") seed = to_size(v);
      else if (k == "diag") diag = to_size(v) != 0;
      else throw ArgError("unknown random parameter: " + k);
    }
    return random_sparse(n_free, p, seed, diag);
  }
  throw ArgError("unknown mask family: '" + name + "'");
}

}  // namespace

// The families gen.cu builds on the device, with the host parser's validation (same messages).
bool bbm::parse_device_family(const std::string& text, uint64_t n_free, bbm::GenSpec& g) {
  std::string name = text, body;
  const size_t open = text.find_first_of("[(");
  if (open != std::string::npos) {
    const char close = text[open] == '[' ? ']' : ')';
    require(text.back() == close, "unbalanced bracket in mask spec: '" + text + "'");
    name = text.substr(0, open);
    body = text.substr(open + 1, text.size() - open - 2);
  }
  g = bbm::GenSpec{};
  g.n = n_free;
  if (name == "causal" || name == "all-ones") {
    require(n_free >= 1, "n must be positive");
    g.family = name == "causal" ? bbm::kGenCausal : bbm::kGenAllOnes;
    return true;
  }
  if (name == "windowed" || name == "dilated" || name == "global") {
    for (const auto& [k, v] : kv(body)) {
      if (k == "w") g.w = to_size(v);
      else if (name == "windowed" && k == "causal") g.causal = to_size(v) != 0;
      else if (name == "dilated" && k == "d") g.d = to_size(v);
      else if (name == "global" && k == "g") g.g = to_size(v);
      else throw ArgError("unknown " + name + " parameter: " + k);
    }
    g.family = name == "windowed" ? bbm::kGenWindowed : name == "dilated" ? bbm::kGenDilated : bbm::kGenGlobal;
    if (g.family == bbm::kGenGlobal) require(g.g <= n_free, "global token count must be <= n");
    require(n_free >= 1, "n must be positive");
    require(g.w < n_free, "window must be < n");
    if (g.family == bbm::kGenDilated) require(g.d >= 1, "dilation must be >= 1");
    return true;
  }
  if (name == "random") {
    for (const auto& [k, v] : kv(body)) {
      if (k == "p") g.p = to_double(v);
      else if (k == "seed") g.seed = to_size(v);
      else if (k == "diag") g.diag = to_size(v) != 0;
      else throw ArgError("unknown random parameter: " + k);
    }
    require(n_free >= 1, "n must be positive");
    require(g.p >= 0.0 && g.p <= 1.0, "density must be in [0, 1]");
    g.family = bbm::kGenRandom;
    return true;
  }
  return false;
}

namespace {

template <class F>
bbm_status guard(F&& f) {
  try {
    f();
    return BBM_OK;
  } catch (const std::invalid_argument& e) {
    bbm::g_last_error = e.what();
    return BBM_ERR_INVALID;
  } catch (const std::exception& e) {
    bbm::g_last_error = e.what();
    return BBM_ERR_INTERNAL;
  }
}

}  // namespace

extern "C" bbm_status bbm_generate(const char* spec, uint64_t n_free, uint64_t* n_out,
                                   uint64_t* words) {
  return guard([&] {
    require(spec != nullptr && n_out != nullptr, "null argument");
    const Bits m = parse_and_generate(spec, n_free);
    *n_out = m.n;
    if (words) std::memcpy(words, m.w.data(), m.w.size() * 8);
  });
}

// generate (generators.hpp:233-438) straight into device memory (d_words: n * ceil(n/64) u64 on
// the current device; NULL queries n). The families of gen.cu run on the device; the others are
// built on the host and uploaded.
extern "C" bbm_status bbm_generate_device(const char* spec, uint64_t n_free, uint64_t* n_out,
                                          uint64_t* d_words, void* stream) {
  return guard([&] {
    require(spec != nullptr && n_out != nullptr, "null argument");
    bbm::GenSpec g;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (bbm::parse_device_family(spec, n_free, g)) {
      *n_out = g.n;
      if (d_words) bbm::launch_generate(g, d_words, s);
      return;
    }
    const Bits m = parse_and_generate(spec, n_free);
    *n_out = m.n;
    if (d_words) {
      BBM_CUDA(cudaMemcpyAsync(d_words, m.w.data(), m.w.size() * 8, cudaMemcpyHostToDevice, s));
      BBM_CUDA(cudaStreamSynchronize(s));
    }
  });
}

extern "C" bbm_status bbm_relabel(const uint64_t* words, uint64_t n, uint64_t seed,
                                  uint64_t* out_words) {
  return guard([&] {
    require(words && out_words && words != out_words, "bad argument");
    std::vector<uint32_t> labels(n);
    std::iota(labels.begin(), labels.end(), 0u);
    std::mt19937_64 gen(seed);
    std::shuffle(labels.begin(), labels.end(), gen);
    const uint64_t wpr = (n + 63) / 64;
    std::memset(out_words, 0, n * wpr * 8);
    for (uint64_t i = 0; i < n; ++i)
      for (uint64_t w = 0; w < wpr; ++w) {
        uint64_t bits = words[i * wpr + w];
        while (bits) {
          const uint64_t j = w * 64 + __builtin_ctzll(bits);
          bits &= bits - 1;
          const uint64_t a = labels[i], b = labels[j];
          out_words[a * wpr + (b >> 6)] |= 1ull << (b & 63);
        }
      }
  });
}

// make_problem's input stream (bench.hpp:320-337, rng.hpp:15-42): per slot q, k, v and d_out,
// each n x d entries uniform in [-1, 1) from one std::mt19937_64(seed), in that order; stored as
// float (the reference's Matrix<float>; its double variant draws the identical doubles).
extern "C" bbm_status bbm_make_problem(uint64_t seed, uint64_t slots, uint64_t n, uint64_t d,
                                       float* q, float* k, float* v, float* d_out) {
  return guard([&] {
    require(q && k && v && d_out, "null argument");
    std::mt19937_64 gen(seed);
    const uint64_t per = n * d;
    for (uint64_t s = 0; s < slots; ++s)
      for (float* dst : {q, k, v, d_out})
        for (uint64_t i = 0; i < per; ++i)
          dst[s * per + i] = static_cast<float>(2.0 * (static_cast<double>(gen() >> 11) * 0x1.0p-53) - 1.0);
  });
}
