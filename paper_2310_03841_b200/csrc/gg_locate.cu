// gg_locate.cu — column checksums of flagged row bands: which 256-column tiles of a
// 128-row band hold the fault a row check flagged (north_star kernel (1): "column
// checksum e^T A plus column sums for tile localisation"; the reference checks rows only,
// SPEC.md:497, and replays the whole layer, guard.py:575-604).
//
// For every band b holding a flagged row (rows 128b .. 128b + 127 of the launch):
//   u_b[k]      = sum_{r in b} X[r, k]                       (e^T X over the band)
//   pred_b[n]   = u_b . W[n, :] + rows_b * bias[n]           (e^T (X W^T + bias))
//   obs_b[n]    = sum_{r in b} C[r, n]                       (e^T C)
//   e_b[n]      = pred_b[n] - obs_b[n]
// A fault at (r, n) that moved row r's check by D moves column n's by the same D, while
// a clean column carries only the rounding of 128 outputs.  Tile (b, t) is marked when a
// column n of it has e_b[n] != 0 (integer operands: exact int64 sums), or (float operands,
// fp64 sums) a non-finite e_b[n] or |e_b[n]| > frac * min over the band's flagged rows with
// a finite d of |d_r - mu| (a fault that made an output Inf / NaN leaves its row's and its
// column's checks non-finite).
//
// Off the clean path (it runs only after a row flag), so plain fp64 / int64 CUDA-core
// arithmetic: three small launches, deterministic folds.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gg_internal.h"

namespace gg {
namespace {

constexpr int LBM = 128;  // rows per band (K1's per-CTA band)
constexpr int LBN = 256;  // columns per tile (K1's pair tile)

__device__ __forceinline__ double ld_real(int dt, const void* p, int64_t i) {
  switch (dt) {
    case GG_BF16: return static_cast<double>(__bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]));
    case GG_F16: return static_cast<double>(__half2float(static_cast<const __half*>(p)[i]));
    case GG_F32: return static_cast<double>(static_cast<const float*>(p)[i]);
    case GG_I32: return static_cast<double>(static_cast<const int32_t*>(p)[i]);
    case GG_I8: return static_cast<double>(static_cast<const int8_t*>(p)[i]);
    default: return 0.0;
  }
}
__device__ __forceinline__ long long ld_int(int dt, const void* p, int64_t i) {
  return dt == GG_I8 ? static_cast<long long>(static_cast<const int8_t*>(p)[i])
                     : static_cast<long long>(static_cast<const int32_t*>(p)[i]);
}

// band threshold: frac * min |d - mu| over the band's flagged rows (float), 0 (integer); -1: no flag
__global__ void locate_bands_kernel(int64_t M, const uint8_t* flags, const void* d, int integer, double mu,
                                    double frac, double* band_thr) {
  __shared__ double s_min[LBM / 32];
  __shared__ int s_any[LBM / 32];
  const int b = blockIdx.x, t = threadIdx.x;
  const int64_t r = static_cast<int64_t>(b) * LBM + t;
  double m = 1.0e308;
  int any = 0;
  if (r < M && flags[r]) {
    any = 1;
    const double dr = integer ? static_cast<double>(static_cast<const long long*>(d)[r])
                              : static_cast<const double*>(d)[r];
    const double g = fabs(dr - mu);
    if (isfinite(g)) m = g;  // a non-finite d: its column's check is non-finite too (marked below)
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
    any |= __shfl_xor_sync(0xffffffffu, any, o);
  }
  if ((t & 31) == 0) {
    s_min[t >> 5] = m;
    s_any[t >> 5] = any;
  }
  __syncthreads();
  if (t == 0) {
    double mm = s_min[0];
    int aa = s_any[0];
    for (int w = 1; w < LBM / 32; ++w) {
      mm = fmin(mm, s_min[w]);
      aa |= s_any[w];
    }
    band_thr[b] = aa ? (integer ? 0.0 : (mm < 1.0e308 ? frac * mm : INFINITY)) : -1.0;
  }
}

// u_b[k] = sum of the band's rows of X (ascending rows): fp64 or int64 bits
__global__ void locate_colsum_x_kernel(int x_dtype, const void* X, int64_t M, int64_t K, int64_t ldx,
                                       const double* band_thr, unsigned long long* u) {
  const int b = blockIdx.y;
  if (band_thr[b] < 0.0) return;
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= K) return;
  const int64_t r0 = static_cast<int64_t>(b) * LBM, r1 = min(M, r0 + LBM);
  if (x_dtype == GG_I8) {
    long long s = 0;
    for (int64_t r = r0; r < r1; ++r) s += ld_int(GG_I8, X, r * ldx + k);
    u[static_cast<int64_t>(b) * K + k] = static_cast<unsigned long long>(s);
  } else {
    double s = 0.0;
    for (int64_t r = r0; r < r1; ++r) s += ld_real(x_dtype, X, r * ldx + k);
    u[static_cast<int64_t>(b) * K + k] = static_cast<unsigned long long>(__double_as_longlong(s));
  }
}

// one warp per column n of band b: e_b[n] = u_b . W[n, :] + rows_b bias[n] - sum_r C[r, n]
__global__ void locate_cols_kernel(int x_dtype, const void* W, int64_t N, int64_t K, int64_t ldw, const void* bias,
                                   int bias_dtype, int c_dtype, const void* C, int64_t M, int64_t ldc,
                                   const double* band_thr, const unsigned long long* u, int n_tiles,
                                   uint8_t* tile_mask, unsigned long long* col_disc) {
  const int b = blockIdx.y;
  const double thr = band_thr[b];
  if (thr < 0.0) return;
  const int lane = threadIdx.x & 31;
  const int64_t n = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (n >= N) return;
  const int64_t r0 = static_cast<int64_t>(b) * LBM, r1 = min(M, r0 + LBM);
  const unsigned long long* ub = u + static_cast<int64_t>(b) * K;
  bool mark;
  unsigned long long bits;
  if (x_dtype == GG_I8) {
    long long p = 0, o = 0;
    for (int64_t k = lane; k < K; k += 32) p += static_cast<long long>(ub[k]) * ld_int(GG_I8, W, n * ldw + k);
    for (int64_t r = r0 + lane; r < r1; r += 32) o += ld_int(GG_I32, C, r * ldc + n);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      p += __shfl_xor_sync(0xffffffffu, p, s);
      o += __shfl_xor_sync(0xffffffffu, o, s);
    }
    const long long bi = bias != nullptr ? ld_int(GG_I32, bias, n) : 0;
    const long long e = p + (r1 - r0) * bi - o;
    mark = e != 0;
    bits = static_cast<unsigned long long>(e);
  } else {
    double p = 0.0, o = 0.0;
    for (int64_t k = lane; k < K; k += 32)
      p = fma(__longlong_as_double(static_cast<long long>(ub[k])), ld_real(x_dtype, W, n * ldw + k), p);
    for (int64_t r = r0 + lane; r < r1; r += 32) o += ld_real(c_dtype, C, r * ldc + n);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      p += __shfl_xor_sync(0xffffffffu, p, s);
      o += __shfl_xor_sync(0xffffffffu, o, s);
    }
    const double bi = bias != nullptr ? ld_real(bias_dtype, bias, n) : 0.0;
    const double e = (p + static_cast<double>(r1 - r0) * bi) - o;
    mark = !isfinite(e) || fabs(e) > thr;
    bits = static_cast<unsigned long long>(__double_as_longlong(e));
  }
  if (lane == 0) {
    if (col_disc != nullptr) col_disc[static_cast<int64_t>(b) * N + n] = bits;
    if (mark) tile_mask[static_cast<int64_t>(b) * n_tiles + n / LBN] = 1;
  }
}

}  // namespace

size_t locate_workspace_bytes(int64_t M, int64_t K) {
  const int64_t m_tiles = (M + LBM - 1) / LBM;
  return static_cast<size_t>(m_tiles) * 8 + static_cast<size_t>(m_tiles * K) * 8 + 256;
}

int launch_locate_tiles(int x_dtype, const void* X, int64_t M, int64_t K, int64_t ldx, const void* W, int64_t N,
                        int64_t ldw, const void* bias, int bias_dtype, int c_dtype, const void* C, int64_t ldc,
                        const uint8_t* flags, const void* d, double mu, double frac, uint8_t* tile_mask,
                        void* col_disc, void* workspace, size_t workspace_bytes, cudaStream_t s) {
  if (M < 1 || N < 1 || K < 1) return fail(GG_EINVAL, "locate_tiles: empty problem");
  if (X == nullptr || W == nullptr || C == nullptr || flags == nullptr || d == nullptr || tile_mask == nullptr ||
      workspace == nullptr)
    return fail(GG_EINVAL, "locate_tiles: null argument");
  if (x_dtype != GG_BF16 && x_dtype != GG_F16 && x_dtype != GG_F32 && x_dtype != GG_I8)
    return fail(GG_EUNSUPPORTED, "locate_tiles: operands must be bf16, fp16, fp32 or int8");
  const bool integer = x_dtype == GG_I8;
  if (integer ? c_dtype != GG_I32 : (c_dtype != GG_BF16 && c_dtype != GG_F16 && c_dtype != GG_F32))
    return fail(GG_EUNSUPPORTED, "locate_tiles: output dtype does not match the operands");
  if (bias != nullptr && (integer ? bias_dtype != GG_I32 : (bias_dtype != GG_F32 && bias_dtype != GG_BF16 &&
                                                            bias_dtype != GG_F16)))
    return fail(GG_EUNSUPPORTED, "locate_tiles: bias dtype");
  if (ldx < K || ldw < K || ldc < N) return fail(GG_EINVAL, "locate_tiles: leading dimensions");
  if (workspace_bytes < locate_workspace_bytes(M, K)) return fail(GG_EINVAL, "locate_tiles: workspace too small");
  if (!(frac > 0.0)) return fail(GG_EINVAL, "locate_tiles: frac must be positive");
  const int64_t m_tiles = (M + LBM - 1) / LBM;
  const int n_tiles = static_cast<int>((N + LBN - 1) / LBN);
  if (m_tiles > 65535) return fail(GG_EUNSUPPORTED, "locate_tiles: more than 65535 bands");
  double* band_thr = static_cast<double*>(workspace);
  unsigned long long* u = reinterpret_cast<unsigned long long*>(
      (reinterpret_cast<uintptr_t>(band_thr + m_tiles) + 255) & ~static_cast<uintptr_t>(255));
  cudaMemsetAsync(tile_mask, 0, static_cast<size_t>(m_tiles) * n_tiles, s);
  locate_bands_kernel<<<static_cast<unsigned>(m_tiles), LBM, 0, s>>>(M, flags, d, integer ? 1 : 0, mu, frac,
                                                                      band_thr);
  locate_colsum_x_kernel<<<dim3(static_cast<unsigned>((K + 255) / 256), static_cast<unsigned>(m_tiles)), 256, 0, s>>>(
      x_dtype, X, M, K, ldx, band_thr, u);
  locate_cols_kernel<<<dim3(static_cast<unsigned>((N + 7) / 8), static_cast<unsigned>(m_tiles)), 256, 0, s>>>(
      x_dtype, W, N, K, ldw, bias, bias_dtype, c_dtype, C, M, ldc, band_thr, u, n_tiles, tile_mask,
      static_cast<unsigned long long*>(col_disc));
  return check_launch("locate_tiles");
}

}  // namespace gg
