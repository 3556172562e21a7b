// pgmres/pattern_hash.hpp — identity of a CSR sparsity pattern for the
// drop-in layers' resident-matrix cache (include/pgmres/dgmres.hpp,
// include/compat + paper_1906_04051_b200/compat/dgmres_device.cpp): a 64-bit
// hash of row_ptr and col_idx, so a cached device matrix is reused only for
// the same pattern (by content, not by the host object's address).
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <thread>
#include <vector>

namespace pgmres {
namespace detail {

inline std::uint64_t hash_span(const std::uint32_t* p, std::size_t n, std::uint64_t seed) {
  constexpr std::uint64_t K1 = 0x9E3779B185EBCA87ull, K2 = 0xC2B2AE3D27D4EB4Full;
  std::uint64_t h = seed ^ (n * K2);
  std::size_t i = 0;
  for (; i + 2 <= n; i += 2) {
    std::uint64_t w = (std::uint64_t(p[i + 1]) << 32) | p[i];
    w *= K2;
    w = (w << 31) | (w >> 33);
    h ^= w * K1;
    h = ((h << 27) | (h >> 37)) * K1 + 0x52DCE729ull;
  }
  if (i < n) {
    h ^= std::uint64_t(p[i]) * K1;
    h = ((h << 27) | (h >> 37)) * K2;
  }
  h ^= h >> 33;
  h *= K2;
  h ^= h >> 29;
  return h;
}

// col_idx is hashed in 16 M-entry chunks over up to 16 host threads (4 GB at
// the largest benchmark mesh); chunk hashes combine in chunk order, so the
// value does not depend on the thread count.
inline std::uint64_t pattern_hash(const std::uint32_t* row_ptr, std::size_t n_rows,
                                  const std::uint32_t* col_idx, std::size_t nnz) {
  constexpr std::size_t CHUNK = std::size_t(1) << 24;
  const std::size_t nchunks = (nnz + CHUNK - 1) / CHUNK;
  std::vector<std::uint64_t> part(nchunks);
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  auto work = [&](unsigned t) {
    for (std::size_t c = t; c < nchunks; c += hw) {
      const std::size_t b = c * CHUNK, e = std::min(nnz, b + CHUNK);
      part[c] = hash_span(col_idx + b, e - b, c);
    }
  };
  if (nchunks > 1 && hw > 1) {
    std::vector<std::thread> team;
    for (unsigned t = 0; t < hw; ++t) team.emplace_back(work, t);
    for (auto& th : team) th.join();
  } else {
    for (unsigned t = 0; t < hw; ++t) work(t);
  }
  std::uint64_t h = hash_span(row_ptr, n_rows + 1, 0x1234567ull);
  for (std::uint64_t v : part) h = (h ^ v) * 0x100000001B3ull + (h >> 17);
  return h;
}

}  // namespace detail
}  // namespace pgmres
