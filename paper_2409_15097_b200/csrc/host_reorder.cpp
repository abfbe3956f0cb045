// host_reorder.cpp — reverse Cuthill-McKee ordering on the host (one-time metadata).
//
// Same permutation as the reference's rcm_order(build_graph(mask)) (reorder.hpp:28-133): the
// graph is the mask pattern symmetrized with self loops dropped; components are taken in
// ascending order of their smallest node, each starts at its minimum-degree node (ties by index),
// BFS frontiers are enqueued by ascending (degree, index), and the whole order is reversed.
//
// Unlike the reference (vector-of-vectors adjacency built by scanning every bit), the graph stays
// a bit matrix: sym = mask | mask^T via 64x64 bit-block transposes, degree = popcount of a row,
// and neighbours come out of a row scan already sorted and de-duplicated.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

#include "../../include/bbm_capi.h"
#include "bbm_internal.h"

namespace {

// In-place transpose of a 64x64 bit block (rows as u64, bit j = column j).
void transpose64(uint64_t a[64]) {
  uint64_t m = 0x00000000FFFFFFFFull;
  for (int j = 32; j != 0; j >>= 1, m ^= (m << j)) {
    for (int k = 0; k < 64; k = ((k | j) + 1) & ~j) {
      const uint64_t t = ((a[k] >> j) ^ a[k | j]) & m;
      a[k] ^= t << j;
      a[k | j] ^= t;
    }
  }
}

struct BitGraph {
  uint64_t n = 0, wpr = 0;
  std::vector<uint64_t> sym;
  std::vector<uint32_t> degree;
};

BitGraph build_bit_graph(const uint64_t* words, uint64_t n) {
  BitGraph g;
  g.n = n;
  g.wpr = (n + 63) / 64;
  const uint64_t wpr = g.wpr;
  g.sym.assign(wpr * 64 * wpr, 0);  // rows padded to a multiple of 64
  for (uint64_t i = 0; i < n; ++i)
    std::memcpy(&g.sym[i * wpr], words + i * wpr, wpr * 8);
  // OR in the transpose, block by block: block (bi, bj) of sym |= transpose(block (bj, bi)).
  uint64_t blk[64];
  std::vector<uint64_t> orig(g.sym);  // transpose source must be the untouched mask
  for (uint64_t bi = 0; bi < wpr; ++bi)
    for (uint64_t bj = 0; bj < wpr; ++bj) {
      bool any = false;
      for (int r = 0; r < 64; ++r) {
        blk[r] = orig[(bj * 64 + r) * wpr + bi];
        any |= blk[r] != 0;
      }
      if (!any) continue;
      transpose64(blk);
      for (int r = 0; r < 64; ++r) g.sym[(bi * 64 + r) * wpr + bj] |= blk[r];
    }
  g.degree.assign(n, 0);
  for (uint64_t i = 0; i < n; ++i) {
    g.sym[i * wpr + (i >> 6)] &= ~(1ull << (i & 63));  // drop self loop
    uint32_t d = 0;
    for (uint64_t w = 0; w < wpr; ++w) d += static_cast<uint32_t>(__builtin_popcountll(g.sym[i * wpr + w]));
    g.degree[i] = d;
  }
  return g;
}

template <class F>
void for_each_neighbor(const BitGraph& g, uint32_t i, F&& f) {
  const uint64_t* row = &g.sym[static_cast<uint64_t>(i) * g.wpr];
  for (uint64_t w = 0; w < g.wpr; ++w) {
    uint64_t bits = row[w];
    while (bits) {
      const uint32_t j = static_cast<uint32_t>(w * 64 + __builtin_ctzll(bits));
      bits &= bits - 1;
      f(j);
    }
  }
}

}  // namespace

extern "C" bbm_status bbm_rcm_order(const uint64_t* words, uint64_t n, uint32_t* forward) {
  try {
    bbm::require(words != nullptr && forward != nullptr, "null argument");
    const BitGraph g = build_bit_graph(words, n);
    std::vector<char> visited(n, 0);
    std::vector<uint32_t> component;
    std::vector<uint32_t> order;
    order.reserve(n);
    auto before = [&](uint32_t a, uint32_t b) {
      return g.degree[a] != g.degree[b] ? g.degree[a] < g.degree[b] : a < b;
    };
    for (uint64_t seed = 0; seed < n; ++seed) {
      if (visited[seed]) continue;
      component.assign(1, static_cast<uint32_t>(seed));
      visited[seed] = 1;
      for (size_t h = 0; h < component.size(); ++h)
        for_each_neighbor(g, component[h], [&](uint32_t nb) {
          if (!visited[nb]) {
            visited[nb] = 1;
            component.push_back(nb);
          }
        });
      uint32_t start = component.front();
      for (uint32_t node : component)
        if (before(node, start)) start = node;
      for (uint32_t node : component) visited[node] = 0;
      const size_t bfs_begin = order.size();
      order.push_back(start);
      visited[start] = 1;
      for (size_t h = bfs_begin; h < order.size(); ++h) {
        const size_t f0 = order.size();
        for_each_neighbor(g, order[h], [&](uint32_t nb) {
          if (!visited[nb]) {
            visited[nb] = 1;
            order.push_back(nb);
          }
        });
        std::sort(order.begin() + f0, order.end(), before);
      }
    }
    std::reverse(order.begin(), order.end());
    std::memcpy(forward, order.data(), n * 4);
    return BBM_OK;
  } catch (const std::invalid_argument& e) {
    bbm::g_last_error = e.what();
    return BBM_ERR_INVALID;
  } catch (const std::exception& e) {
    bbm::g_last_error = e.what();
    return BBM_ERR_INTERNAL;
  }
}

extern "C" bbm_status bbm_bandwidth(const uint64_t* words, uint64_t n, uint64_t* bandwidth) {
  // reorder.hpp:137-153: max |i - j| over set entries
  if (!words || !bandwidth) {
    bbm::g_last_error = "null argument";
    return BBM_ERR_INVALID;
  }
  const uint64_t wpr = (n + 63) / 64;
  uint64_t bw = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t* row = words + i * wpr;
    uint64_t first = n, last = 0;
    for (uint64_t w = 0; w < wpr; ++w)
      if (row[w]) {
        first = w * 64 + __builtin_ctzll(row[w]);
        break;
      }
    if (first == n) continue;
    for (uint64_t w = wpr; w-- > 0;)
      if (row[w]) {
        last = w * 64 + 63 - __builtin_clzll(row[w]);
        break;
      }
    if (first < i) bw = std::max(bw, i - first);
    if (last > i) bw = std::max(bw, last - i);
  }
  *bandwidth = bw;
  return BBM_OK;
}

extern "C" bbm_status bbm_graph_csr(const uint64_t* words, uint64_t n, uint64_t* offsets,
                                    uint32_t* neighbors) {
  // build_graph (reorder.hpp:28-49): symmetrized pattern, self loops dropped, neighbours sorted
  try {
    bbm::require(words != nullptr && offsets != nullptr, "null argument");
    const BitGraph g = build_bit_graph(words, n);
    offsets[0] = 0;
    for (uint64_t i = 0; i < n; ++i) offsets[i + 1] = offsets[i] + g.degree[i];
    if (neighbors)
      for (uint64_t i = 0; i < n; ++i) {
        uint64_t at = offsets[i];
        for_each_neighbor(g, static_cast<uint32_t>(i), [&](uint32_t j) { neighbors[at++] = j; });
      }
    return BBM_OK;
  } catch (const std::invalid_argument& e) {
    bbm::g_last_error = e.what();
    return BBM_ERR_INVALID;
  } catch (const std::exception& e) {
    bbm::g_last_error = e.what();
    return BBM_ERR_INTERNAL;
  }
}
