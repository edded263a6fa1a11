// Shared host-side analysis of the contraction family (FFMA and tensor-core
// templates): operand roles, dim groups and the additive offset tables.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <numeric>
#include <vector>

#include "../plan.hpp"

namespace mdhb {
namespace ctr {

struct Groups {
  int a_buf = 0, b_buf = 1;
  Linear la, lb, lc;
  std::vector<int> Md, Nd, Kd;  // outer -> inner
};

inline int64_t prod_sizes(const MdHom& e, const std::vector<int>& dims) {
  int64_t p = 1;
  for (int d : dims) p *= e.sizes[static_cast<size_t>(d)];
  return p;
}

// Enumerates the box `ext` (row-major over dims) and returns sum_d c[dims[t]] * l_t * scale_t
inline std::vector<int64_t> box_offsets(const std::vector<int>& dims, const std::vector<int64_t>& ext,
                                 const std::vector<int64_t>& coef, const std::vector<int64_t>& scale) {
  int64_t n = 1;
  for (int64_t x : ext) n *= x;
  std::vector<int64_t> out(static_cast<size_t>(n), 0);
  std::vector<int64_t> l(dims.size(), 0);
  for (int64_t t = 0; t < n; ++t) {
    int64_t o = 0;
    for (size_t q = 0; q < dims.size(); ++q) o += coef[static_cast<size_t>(dims[q])] * l[q] * scale[q];
    out[static_cast<size_t>(t)] = o;
    for (int q = static_cast<int>(dims.size()) - 1; q >= 0; --q) {
      if (++l[static_cast<size_t>(q)] < ext[static_cast<size_t>(q)]) break;
      l[static_cast<size_t>(q)] = 0;
    }
  }
  return out;
}

// Splits `target` cells over the dims' extents (inner -> outer) with gcds;
// empty when the box cannot be formed exactly.
inline std::vector<int64_t> factor_box(const MdHom& e, const std::vector<int>& dims, int64_t target) {
  std::vector<int64_t> t(dims.size(), 1);
  int64_t rem = target;
  for (int q = static_cast<int>(dims.size()) - 1; q >= 0 && rem > 1; --q) {
    int64_t g = std::gcd(e.sizes[static_cast<size_t>(dims[static_cast<size_t>(q)])], rem);
    t[static_cast<size_t>(q)] = g;
    rem /= g;
  }
  if (rem != 1) return {};
  return t;
}

// Tensor-core (tcgen05, TF32) instance of the contraction template for the
// same groups; nullptr (and the reason in *why) when the operands cannot be
// described as TMA boxes -- the caller then keeps the FFMA template.
std::unique_ptr<Routine> make_tc_contraction(const Problem& p, const Groups& g, const Config* cfg, Config* cfg_out,
                                             std::string* why);

// The tensor-core GEMM template's instances for a MatMul-shaped md_hom, as
// canonical Table-1 configurations (empty for other shapes).
std::vector<Config> tc_space(const Problem& p, const Groups& g);
// The tensor-core instance a configuration instantiates, as its canonical
// configuration (false: not MatMul-shaped / FFMA; throws Unsupported when
// the configuration is outside the template).
bool tc_project(const Problem& p, const Groups& g, const Config& c, Config* canon);

// Tensor-core instance for NHWC convolutions (MCC): one input patch per
// 32-channel chunk, all R*S taps issued from it through shifted descriptors
// (kernels/tc_conv.cu).  nullptr when the md_hom is not such a convolution.
std::unique_ptr<Routine> make_tc_conv(const Problem& p, const Groups& g, std::string* why);

// NHWC convolution read off an md_hom (MCC's views): O[n][p][q][k] =
// sum_{r,s,c} I[n][p+r][q+s][c] * F[k][r][s][c].  Extents are the views'
// inferred extents; strides are row-major over them.
struct ConvShape {
  int ib = -1, fb = -1;                 // input / filter buffers
  int N = 0, P = 0, Q = 0, K = 0, R = 0, S = 0, C = 0;
  int64_t H = 0, W = 0;                 // input rows / columns
  std::vector<int64_t> oe;              // output extents [N][P][Q][K]
};
// True when buffers (ib, fb) form such a convolution (kernels/tc_conv.cu).
bool nhwc_conv_shape(const Problem& p, int ib, int fb, ConvShape* s, std::string* why);

// FP32 FFMA instance for NHWC convolutions with K = 64, 3x3 taps, Q % 8 == 0
// (kernels/ffma_conv.cu); nullptr when the md_hom is not such a convolution.
std::unique_ptr<Routine> make_ffma_conv(const Problem& p, const Groups& g, std::string* why);

}  // namespace ctr
}  // namespace mdhb
