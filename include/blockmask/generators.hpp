// blockmask/generators.hpp — the reference's mask families (proj/include/blockmask/
// generators.hpp:22-183) as host fixtures, produced by libbbm's generator (bbm_generate) so the
// masks are bit-identical to the reference's (tests/test_host.py pins them against golden
// vectors generated from the reference itself).
#pragma once

#include <cstdint>
#include <cstdio>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "blockmask/device.hpp"
#include "blockmask/mask.hpp"

namespace blockmask {

/// MaskSpec grammar (generators.hpp:364-438): e.g. "causal", "medusa[4;4;4;4]",
/// "global(w=512;g=128)"; families with a free size take n.
inline Mask generate_spec(const std::string& spec, std::size_t n = 0) {
    std::uint64_t size = 0;
    device::check(bbm_generate(spec.c_str(), n, &size, nullptr), "generate");
    Mask m(size);
    device::check(bbm_generate(spec.c_str(), n, &size, m.words()), "generate");
    return m;
}

namespace detail {
inline std::string join(std::span<const std::size_t> v) {
    std::string s;
    for (std::size_t i = 0; i < v.size(); ++i) s += (i ? ";" : "") + std::to_string(v[i]);
    return s;
}
}  // namespace detail

inline std::size_t medusa_size(std::span<const std::size_t> candidates) {
    require(!candidates.empty(), "medusa candidate list must be non-empty");
    std::size_t total = 0, level = 1;
    for (std::size_t c : candidates) {
        level *= c;
        total += level;
    }
    return total;
}

inline Mask gen_medusa(std::span<const std::size_t> c) { return generate_spec("medusa[" + detail::join(c) + "]"); }
inline Mask gen_causal(std::size_t n) { return generate_spec("causal", n); }
inline Mask gen_all_ones(std::size_t n) { return generate_spec("all-ones", n); }
inline Mask gen_packed_sequential(std::span<const std::size_t> lengths) {
    return generate_spec("packed-seq[" + detail::join(lengths) + "]");
}
inline Mask gen_packed_input_bidirectional(std::span<const std::pair<std::size_t, std::size_t>> segs) {
    std::string s = "packed-bidir[";
    for (std::size_t i = 0; i < segs.size(); ++i)
        s += (i ? ";" : "") + std::to_string(segs[i].first) + ":" + std::to_string(segs[i].second);
    return generate_spec(s + "]");
}
inline Mask gen_longformer_windowed(std::size_t n, std::size_t window, bool causal = false) {
    return generate_spec("windowed(w=" + std::to_string(window) + (causal ? ";causal=1)" : ")"), n);
}
inline Mask gen_longformer_dilated(std::size_t n, std::size_t window, std::size_t dilation) {
    return generate_spec("dilated(w=" + std::to_string(window) + ";d=" + std::to_string(dilation) + ")", n);
}
inline Mask gen_longformer_global(std::size_t n, std::size_t window, std::size_t global_count) {
    return generate_spec("global(w=" + std::to_string(window) + ";g=" + std::to_string(global_count) + ")", n);
}
inline Mask gen_random_sparse(std::size_t n, double density, std::uint64_t seed, bool force_diagonal = true) {
    char p[64];
    std::snprintf(p, sizeof p, "%.17g", density);
    return generate_spec(std::string("random(p=") + p + ";seed=" + std::to_string(seed) +
                             (force_diagonal ? ")" : ";diag=0)"),
                         n);
}

}  // namespace blockmask
