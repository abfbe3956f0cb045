// blockmask/generators.hpp — the reference's mask families (proj/include/blockmask/
// generators.hpp:22-183) as host fixtures, produced by libbbm's generator (bbm_generate) so the
// masks are bit-identical to the reference's (tests/test_host.py pins them against golden
// vectors generated from the reference itself).
#pragma once

#include <cstdint>
#include <cstdio>
#include <random>  // the reference's header brings std::mt19937_64 along (callers rely on it)
#include <sstream>
#include <span>
#include <string>
#include <type_traits>
#include <utility>
#include <variant>
#include <vector>

#include "blockmask/device.hpp"
#include "blockmask/mask.hpp"
#include "blockmask/mask_io.hpp"

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

/// MaskSpec (generators.hpp:190-438): a tagged description of a mask family with the
/// reference's string grammar. parse() / to_string() round-trip; generate() builds the mask
/// through libbbm (bit-identical to the reference's generators).
struct MaskSpec {
    struct Causal { std::size_t n = 0; };
    struct AllOnes { std::size_t n = 0; };
    struct Medusa { std::vector<std::size_t> candidates; };
    struct PackedSequential { std::vector<std::size_t> lengths; };
    struct PackedInputBidirectional { std::vector<std::pair<std::size_t, std::size_t>> segments; };
    struct Windowed { std::size_t n = 0; std::size_t window = 0; bool causal = false; };
    struct Dilated { std::size_t n = 0; std::size_t window = 0; std::size_t dilation = 1; };
    struct Global { std::size_t n = 0; std::size_t window = 0; std::size_t global_count = 0; };
    struct RandomSparse {
        std::size_t n = 0;
        double density = 0.0;
        std::uint64_t seed = 0;
        bool force_diagonal = true;
    };
    struct File { std::string path; };

    std::variant<Causal, AllOnes, Medusa, PackedSequential, PackedInputBidirectional, Windowed, Dilated,
                 Global, RandomSparse, File>
        value{Causal{}};

    /// Families whose size is a free parameter (set by with_n).
    bool has_free_n() const {
        return std::visit([](const auto& v) { return requires { v.n; }; }, value);
    }

    MaskSpec with_n(std::size_t n) const {
        MaskSpec out = *this;
        std::visit([n](auto& v) {
            if constexpr (requires { v.n; }) v.n = n;
        }, out.value);
        return out;
    }

    std::string to_string() const;
    static MaskSpec parse(const std::string& text);
};

namespace detail {
inline std::vector<std::string> split_on(const std::string& s, char sep) {
    std::vector<std::string> out(1);
    for (char c : s) {
        if (c == sep) out.emplace_back();
        else out.back() += c;
    }
    return out;
}
inline std::size_t spec_size(const std::string& t) {
    require(!t.empty() && t.find_first_not_of("0123456789") == std::string::npos,
            "bad integer in mask spec: '" + t + "'");
    return static_cast<std::size_t>(std::stoull(t));
}
inline double spec_double(const std::string& t) {
    std::size_t used = 0;
    double v = 0.0;
    try {
        v = std::stod(t, &used);
    } catch (const std::exception&) {
        throw std::invalid_argument("bad number in mask spec: '" + t + "'");
    }
    require(used == t.size(), "bad number in mask spec: '" + t + "'");
    return v;
}
// the reference's names for the same helpers (generators.hpp:276-308; its bench.hpp parses CSV
// rows with them)
inline std::vector<std::string> split(const std::string& text, char sep) { return split_on(text, sep); }
inline std::size_t parse_size(const std::string& text) { return spec_size(text); }
inline double parse_double(const std::string& text) { return spec_double(text); }
// key=value;key=value -> visits (key, value), rejecting items without '='
template <class F>
void spec_params(const std::string& body, F&& on) {
    if (body.empty()) return;
    for (const std::string& item : split_on(body, ';')) {
        const std::size_t eq = item.find('=');
        require(eq != std::string::npos, "expected key=value in mask spec: '" + item + "'");
        on(item.substr(0, eq), item.substr(eq + 1));
    }
}
}  // namespace detail

inline std::string MaskSpec::to_string() const {
    std::ostringstream o;
    auto sizes = [&](const std::vector<std::size_t>& xs) {
        for (std::size_t i = 0; i < xs.size(); ++i) o << (i ? ";" : "") << xs[i];
    };
    std::visit([&](const auto& v) {
        using V = std::decay_t<decltype(v)>;
        if constexpr (std::is_same_v<V, Causal>) o << "causal";
        else if constexpr (std::is_same_v<V, AllOnes>) o << "all-ones";
        else if constexpr (std::is_same_v<V, Medusa>) { o << "medusa["; sizes(v.candidates); o << "]"; }
        else if constexpr (std::is_same_v<V, PackedSequential>) { o << "packed-seq["; sizes(v.lengths); o << "]"; }
        else if constexpr (std::is_same_v<V, PackedInputBidirectional>) {
            o << "packed-bidir[";
            for (std::size_t i = 0; i < v.segments.size(); ++i)
                o << (i ? ";" : "") << v.segments[i].first << ':' << v.segments[i].second;
            o << "]";
        } else if constexpr (std::is_same_v<V, Windowed>) o << "windowed(w=" << v.window << (v.causal ? ";causal=1" : "") << ")";
        else if constexpr (std::is_same_v<V, Dilated>) o << "dilated(w=" << v.window << ";d=" << v.dilation << ")";
        else if constexpr (std::is_same_v<V, Global>) o << "global(w=" << v.window << ";g=" << v.global_count << ")";
        else if constexpr (std::is_same_v<V, RandomSparse>)
            o << "random(p=" << v.density << ";seed=" << v.seed << (v.force_diagonal ? "" : ";diag=0") << ")";
        else o << "file:" << v.path;
    }, value);
    return o.str();
}

inline MaskSpec MaskSpec::parse(const std::string& text) {
    MaskSpec spec;
    if (text.rfind("file:", 0) == 0) {
        spec.value = File{text.substr(5)};
        return spec;
    }
    std::string name = text, body;
    const std::size_t open = text.find_first_of("[(");
    if (open != std::string::npos) {
        const char close = text[open] == '[' ? ']' : ')';
        require(text.back() == close, "unbalanced bracket in mask spec: '" + text + "'");
        name = text.substr(0, open);
        body = text.substr(open + 1, text.size() - open - 2);
    }
    auto unknown = [&](const std::string& key) {
        throw std::invalid_argument("unknown " + name + " parameter: " + key);
    };
    if (name == "causal") spec.value = Causal{};
    else if (name == "all-ones") spec.value = AllOnes{};
    else if (name == "medusa" || name == "packed-seq") {
        std::vector<std::size_t> xs;
        for (const std::string& t : detail::split_on(body, ';')) xs.push_back(detail::spec_size(t));
        if (name == "medusa") spec.value = Medusa{std::move(xs)};
        else spec.value = PackedSequential{std::move(xs)};
    } else if (name == "packed-bidir") {
        PackedInputBidirectional pb;
        for (const std::string& t : detail::split_on(body, ';')) {
            const auto io = detail::split_on(t, ':');
            require(io.size() == 2, "expected in:out segment in mask spec: '" + t + "'");
            pb.segments.emplace_back(detail::spec_size(io[0]), detail::spec_size(io[1]));
        }
        spec.value = std::move(pb);
    } else if (name == "windowed") {
        Windowed w;
        detail::spec_params(body, [&](const std::string& k, const std::string& v) {
            if (k == "w") w.window = detail::spec_size(v);
            else if (k == "causal") w.causal = detail::spec_size(v) != 0;
            else unknown(k);
        });
        spec.value = w;
    } else if (name == "dilated") {
        Dilated d;
        detail::spec_params(body, [&](const std::string& k, const std::string& v) {
            if (k == "w") d.window = detail::spec_size(v);
            else if (k == "d") d.dilation = detail::spec_size(v);
            else unknown(k);
        });
        spec.value = d;
    } else if (name == "global") {
        Global g;
        detail::spec_params(body, [&](const std::string& k, const std::string& v) {
            if (k == "w") g.window = detail::spec_size(v);
            else if (k == "g") g.global_count = detail::spec_size(v);
            else unknown(k);
        });
        spec.value = g;
    } else if (name == "random") {
        RandomSparse r;
        detail::spec_params(body, [&](const std::string& k, const std::string& v) {
            if (k == "p") r.density = detail::spec_double(v);
            else if (k == "seed") r.seed = detail::spec_size(v);
            else if (k == "diag") r.force_diagonal = detail::spec_size(v) != 0;
            else unknown(k);
        });
        spec.value = r;
    } else {
        throw std::invalid_argument("unknown mask family: '" + name + "'");
    }
    return spec;
}

/// generate (generators.hpp:233-262): the family's mask; file specs read a BBMK file.
inline Mask generate(const MaskSpec& spec) {
    if (const auto* f = std::get_if<MaskSpec::File>(&spec.value)) return read_mask(f->path);
    const std::size_t n = std::visit([](const auto& v) -> std::size_t {
        if constexpr (requires { v.n; }) return v.n;
        else return 0;
    }, spec.value);
    if (const auto* r = std::get_if<MaskSpec::RandomSparse>(&spec.value))  // full double precision
        return gen_random_sparse(r->n, r->density, r->seed, r->force_diagonal);
    return generate_spec(spec.to_string(), n);
}

}  // namespace blockmask
