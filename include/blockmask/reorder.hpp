// blockmask/reorder.hpp — drop-in for the reference's RCM reordering (proj/include/blockmask/
// reorder.hpp:21-189). The ordering itself is one-time host metadata (as the north star asks);
// the data movement runs on the device:
//
//   build_graph    (reorder.hpp:28-49)    -> bbm_graph_csr (bit-matrix symmetrization, host)
//   rcm_order      (reorder.hpp:85-133)   -> bbm_rcm_order (host, identical tie-breaking)
//   bandwidth      (reorder.hpp:137-153)  -> bbm_bandwidth (host)
//   permute_mask   (reorder.hpp:156-163)  -> bbm_permute_mask_host (device kernel)
//   permute_rows / unpermute_rows (reorder.hpp:167-189) -> bbm_permute_rows_host (device kernel)
#pragma once

#include <cstdint>
#include <vector>

#include "blockmask/device.hpp"
#include "blockmask/mask.hpp"
#include "blockmask/matrix.hpp"

namespace blockmask {

/// Undirected pattern: edge i-j iff mask(i,j) or mask(j,i), no self loops, sorted neighbours.
struct SparsityGraph {
    std::size_t n_nodes = 0;
    std::vector<std::vector<std::uint32_t>> adjacency;

    std::size_t degree(std::size_t i) const { return adjacency[i].size(); }
};

inline SparsityGraph build_graph(const Mask& mask) {
    const std::size_t n = mask.size();
    SparsityGraph g{n, std::vector<std::vector<std::uint32_t>>(n)};
    if (n == 0) return g;
    std::vector<std::uint64_t> off(n + 1);
    device::check(bbm_graph_csr(mask.words(), n, off.data(), nullptr), "build_graph");
    std::vector<std::uint32_t> nb(off[n]);
    device::check(bbm_graph_csr(mask.words(), n, off.data(), nb.data()), "build_graph");
    for (std::size_t i = 0; i < n; ++i) g.adjacency[i].assign(nb.begin() + off[i], nb.begin() + off[i + 1]);
    return g;
}

/// forward maps new -> old, inverse old -> new (reorder.hpp:53-79).
struct Permutation {
    std::vector<std::uint32_t> forward;
    std::vector<std::uint32_t> inverse;

    static Permutation from_forward(std::vector<std::uint32_t> fwd) {
        Permutation p;
        p.inverse.assign(fwd.size(), 0);
        std::vector<char> seen(fwd.size(), 0);
        for (std::size_t a = 0; a < fwd.size(); ++a) {
            require(fwd[a] < fwd.size() && !seen[fwd[a]], "forward map is not a bijection");
            seen[fwd[a]] = 1;
            p.inverse[fwd[a]] = static_cast<std::uint32_t>(a);
        }
        p.forward = std::move(fwd);
        return p;
    }
    static Permutation identity(std::size_t n) {
        std::vector<std::uint32_t> f(n);
        for (std::size_t i = 0; i < n; ++i) f[i] = static_cast<std::uint32_t>(i);
        return from_forward(std::move(f));
    }
    std::size_t size() const { return forward.size(); }
    friend bool operator==(const Permutation&, const Permutation&) = default;
};

/// RCM over the graph. The graph is symmetric without self loops, so its adjacency bit matrix
/// is a mask whose build_graph is the graph itself; libbbm orders that.
inline Permutation rcm_order(const SparsityGraph& g) {
    const std::size_t n = g.n_nodes;
    if (n == 0) return Permutation{};
    Mask adj(n);
    for (std::size_t i = 0; i < n; ++i)
        for (std::uint32_t j : g.adjacency[i]) adj.set(i, j, true);
    std::vector<std::uint32_t> fwd(n);
    device::check(bbm_rcm_order(adj.words(), n, fwd.data()), "rcm_order");
    return Permutation::from_forward(std::move(fwd));
}

inline std::size_t bandwidth(const Mask& mask) {
    if (mask.size() == 0) return 0;
    std::uint64_t bw = 0;
    device::check(bbm_bandwidth(mask.words(), mask.size(), &bw), "bandwidth");
    return static_cast<std::size_t>(bw);
}

inline Mask permute_mask(const Mask& mask, const Permutation& perm) {
    require(perm.size() == mask.size(), "permutation length must match mask size");
    Mask out(mask.size());
    if (mask.size() == 0) return out;
    device::check(bbm_permute_mask_host(mask.words(), out.words(), perm.forward.data(), mask.size(),
                                        device::default_device()),
                  "permute_mask");
    return out;
}

namespace detail {
template <typename T>
Matrix<T> move_rows(const Matrix<T>& m, const Permutation& perm, int inverse) {
    require(perm.size() == m.rows(), "permutation length must match row count");
    Matrix<T> out(m.rows(), m.cols());
    if (m.size() == 0) return out;
    device::check(bbm_permute_rows_host(m.data(), out.data(), perm.forward.data(), 1, m.rows(),
                                        m.cols() * sizeof(T), inverse, device::default_device()),
                  inverse ? "unpermute_rows" : "permute_rows");
    return out;
}
}  // namespace detail

/// out.row(a) = m.row(forward[a])
template <typename T>
Matrix<T> permute_rows(const Matrix<T>& m, const Permutation& perm) {
    return detail::move_rows(m, perm, 0);
}

/// out.row(forward[a]) = m.row(a)
template <typename T>
Matrix<T> unpermute_rows(const Matrix<T>& m, const Permutation& perm) {
    return detail::move_rows(m, perm, 1);
}

}  // namespace blockmask
