// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the reference's own tt_config.cpp, which is
// compiled where it lies (/root/reference/proj/core/src/tt_config.cpp, the
// only hot-path translation unit that needs no Eigen) into
// oracle/_ref/libttref.so by oracle/Makefile.  tests/test_ref_pin.py uses it
// to pin the C restatement's index math bit-exactly against the reference.
// tt_embedding.cpp and autodiff.cpp need Eigen3, which is absent from this
// image (no network), so they are not built.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "ttgnn/tt_config.hpp"

using ttgnn::index_t;

namespace {
ttgnn::TTConfig make(int64_t M, int64_t N, int32_t d, const int64_t* m, const int64_t* n,
                     const int64_t* R) {
  return ttgnn::plan_factorization(M, N, std::vector<index_t>(m, m + d),
                                   std::vector<index_t>(n, n + d),
                                   std::vector<index_t>(R, R + d + 1));
}
}  // namespace

extern "C" {

// 0 = valid, 1 = std::invalid_argument from TTConfig::validate.
int ref_validate(int64_t M, int64_t N, int32_t d, const int64_t* m, const int64_t* n,
                 const int64_t* R) {
  try { make(M, N, d, m, n, R); return 0; } catch (const std::invalid_argument&) { return 1; }
}

int64_t ref_count_params(int64_t M, int64_t N, int32_t d, const int64_t* m, const int64_t* n,
                         const int64_t* R) {
  return ttgnn::count_params(make(M, N, d, m, n, R));
}

// Digits for rows[0..count); returns -1, or the first row that threw
// std::out_of_range.
int64_t ref_index_to_coordinate(int64_t M, int64_t N, int32_t d, const int64_t* m,
                                const int64_t* n, const int64_t* R, const int64_t* rows,
                                int64_t count, int64_t* parts) {
  auto cfg = make(M, N, d, m, n, R);
  for (int64_t b = 0; b < count; ++b) {
    try {
      auto c = ttgnn::index_to_coordinate(cfg, rows[b]);
      for (int32_t k = 0; k < d; ++k) parts[b * d + k] = c.parts[k];
    } catch (const std::out_of_range&) {
      return b;
    }
  }
  return -1;
}

int64_t ref_coordinate_to_index(int64_t M, int64_t N, int32_t d, const int64_t* m,
                                const int64_t* n, const int64_t* R, const int64_t* parts) {
  auto cfg = make(M, N, d, m, n, R);
  ttgnn::RowCoordinate c;
  c.parts.assign(parts, parts + d);
  try { return ttgnn::coordinate_to_index(cfg, c); } catch (...) { return -1; }
}

// Auto planner (tt_config.cpp:144-160): writes m, n (d each).
int ref_plan_auto(int64_t M, int64_t N, int32_t d, const int64_t* R, int ortho_friendly,
                  int64_t* m_out, int64_t* n_out) {
  try {
    auto cfg = ttgnn::plan_factorization(M, N, d, std::vector<index_t>(R, R + d + 1),
                                         ortho_friendly != 0);
    for (int32_t k = 0; k < d; ++k) { m_out[k] = cfg.row_factors[k]; n_out[k] = cfg.col_factors[k]; }
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

}  // extern "C"
