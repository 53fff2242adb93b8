// gg_vit.cu — the transformer glue between the protected GEMMs of the ViT /
// Swin forward (unprotected: only the Linear layers carry
// checksums).  HBM-bound elementwise / row work, one pass each:
//
//   gg_add_layernorm   h <- h + y (residual update, optional) and a = LN(h) * gamma + beta
//                      in one read of h, y and one write of h, a (fp32 statistics)
//
// One warp per row, 16-byte vector accesses, the row held in registers
// between the statistics and the normalisation (two-pass mean / variance).
#include <algorithm>

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gg_internal.h"

namespace gg {
namespace {

template <typename T>
struct Vec;  // 16 bytes of T
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static void load(const void* p, float (&v)[8]) {
    const uint4 u = *static_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
  __device__ static void store(void* p, const float (&v)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 b = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<const uint32_t*>(&b);
    }
    *static_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <>
struct Vec<__half> {
  static constexpr int N = 8;
  __device__ static void load(const void* p, float (&v)[8]) {
    const uint4 u = *static_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  }
  __device__ static void store(void* p, const float (&v)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<const uint32_t*>(&h);
    }
    *static_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <>
struct Vec<float> {
  static constexpr int N = 4;
  __device__ static void load(const void* p, float (&v)[4]) {
    const float4 u = *static_cast<const float4*>(p);
    v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
  }
  __device__ static void store(void* p, const float (&v)[4]) {
    *static_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};

// 256-thread blocks resident per SM for a lane holding `floats` row values (register budget)
constexpr int ln_min_blocks(int floats) { return floats <= 24 ? 4 : floats <= 32 ? 3 : floats <= 48 ? 2 : 1; }

// CH = 16-byte chunks per lane (D = 32 * CH * Vec::N); one warp per row.  The rows in flight
// hide HBM latency, and those come from resident warps, so the register budget is capped for
// four 256-thread blocks per SM at D = 768: the predicted-sum variant otherwise took more than
// 64 registers, three blocks, and ran 25% slower (two or four rows per warp sharing the affine
// parameter loads measured slower still).
// EMB (the ViT embedding, emb_T tokens per image): row (b, t) of the residual stream is
// cls + pos[0] for t = 0 and e[b, t - 1] + pos[t] otherwise (h = e, y = pos, cls below), the
// sum rounded to T like torch's add -- the patch embedding's position add, class token and
// first layer norm in one pass.
template <typename T, int CH, bool PRED, bool EMB = false>
// h_out may alias h (in-place residual update): neither is __restrict__.
__global__ void __launch_bounds__(256, ln_min_blocks(CH * Vec<T>::N)) add_layernorm_kernel(const T* h, const T* __restrict__ y, int64_t rows, int D,
                                                            const float* __restrict__ gamma,
                                                            const float* __restrict__ beta, float eps, T* h_out,
                                                            T* __restrict__ ln_out, const float* __restrict__ w_pred,
                                                            unsigned long long* __restrict__ pred_out,
                                                            const T* __restrict__ cls = nullptr, int emb_T = 0) {
  constexpr int V = Vec<T>::N;
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const T* hr = h + row * D;
  const T* yr = y + row * D;
  if constexpr (EMB) {
    const int64_t b = row / emb_T, t = row - b * emb_T;
    hr = t == 0 ? cls : h + (b * (emb_T - 1) + t - 1) * D;
    yr = y + t * D;
  }
  float v[CH][V];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int col = (c * 32 + lane) * V;
    Vec<T>::load(hr + col, v[c]);
    if (y != nullptr) {
      float t[V];
      Vec<T>::load(yr + col, t);
#pragma unroll
      for (int i = 0; i < V; ++i) v[c][i] += t[i];
      uint4 packed;  // the stored (rounded) residual is what LN sees
      Vec<T>::store(&packed, v[c]);
      Vec<T>::load(&packed, v[c]);
      *reinterpret_cast<uint4*>(h_out + row * D + col) = packed;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int i = 0; i < V; ++i) s += v[c][i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / static_cast<float>(D);
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float dv = v[c][i] - mean;
      q += dv * dv;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rstd = rsqrtf(q / static_cast<float>(D) + eps);
  float p = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int col = (c * 32 + lane) * V;
    float gm[V], bt[V], o[V];
#pragma unroll
    for (int i = 0; i < V; i += 4) {  // 16-byte loads of the (L1-resident) affine parameters
      const float4 g4 = __ldg(reinterpret_cast<const float4*>(gamma + col + i));
      const float4 b4 = __ldg(reinterpret_cast<const float4*>(beta + col + i));
      gm[i] = g4.x; gm[i + 1] = g4.y; gm[i + 2] = g4.z; gm[i + 3] = g4.w;
      bt[i] = b4.x; bt[i + 1] = b4.y; bt[i + 2] = b4.z; bt[i + 3] = b4.w;
    }
#pragma unroll
    for (int i = 0; i < V; ++i) o[i] = fmaf((v[c][i] - mean) * rstd, gm[i], bt[i]);
    if constexpr (PRED) {  // the consumer's predicted sum over the stored (rounded) values
      uint4 packed;
      Vec<T>::store(&packed, o);
      Vec<T>::load(&packed, o);
      *reinterpret_cast<uint4*>(ln_out + row * D + col) = packed;
#pragma unroll
      for (int i = 0; i < V; i += 4) {
        const float4 w4 = __ldg(reinterpret_cast<const float4*>(w_pred + col + i));
        p = fmaf(o[i], w4.x, p);
        p = fmaf(o[i + 1], w4.y, p);
        p = fmaf(o[i + 2], w4.z, p);
        p = fmaf(o[i + 3], w4.w, p);
      }
    } else {
      Vec<T>::store(ln_out + row * D + col, o);
    }
  }
  if constexpr (PRED) {
    // fp32 chain of D/32 products per lane and a fixed butterfly over the lanes (deterministic;
    // every lane ends with the same bits since a + b is commutative): error <= (D/32 + 5) 2^-24
    // sum |x w|, inside the fused check's 2^-19 sum |terms| bound for D <= 4096
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
    if (lane == 0) pred_out[row] = static_cast<unsigned long long>(__float_as_uint(p));  // (hi, lo = 0)
  }
}

// The plain layer norm (no residual add, no predicted sums: the ViT's norms once the GEMMs
// store the residual update) as a persistent grid: each warp walks rows row0, row0 + stride, ...,
// keeps its lanes' affine parameters in registers (loaded once instead of once per row: five
// times the row's own bytes of L1 traffic) and loads its next row before reducing the current
// one.  Same sums in the same order as add_layernorm_kernel (identical bytes).  ViT-B b256
// (50432 x 768 bf16): 47.5 -> 43 us, against 33.3 us for a plain copy of the same bytes; ViT-L
// width (1024, no prefetch: 56 bytes of spill for the affine registers): 79 -> 52.5 us
// (tools/ab_ln.py, tools/ln_ref.py).  Slower alternatives measured: more resident warps with the
// row kept packed (54 / 63 us at six / eight blocks per SM), rows staged through a per-warp TMA
// ring in shared memory (50-63 us for 4-12 rows in flight per warp).
#ifndef GG_LN_STREAM_BPS
#define GG_LN_STREAM_BPS 2  // resident 256-thread blocks per SM (the affine registers: 76 per thread)
#endif
template <typename T, int CH, bool PRED>
__global__ void __launch_bounds__(256, GG_LN_STREAM_BPS) layernorm_stream_kernel(const T* __restrict__ h, int64_t rows,
                                                                                 int D, const float* __restrict__ gamma,
                                                                                 const float* __restrict__ beta,
                                                                                 float eps, T* __restrict__ ln_out,
                                                                                 const float* __restrict__ w_pred,
                                                                                 unsigned long long* __restrict__ pred_out) {
  constexpr int V = Vec<T>::N;
  const int lane = threadIdx.x & 31;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  constexpr bool PF = CH <= 3;  // prefetch the next row (wider rows: the registers go to the affine parameters)
  uint4 cur[CH], nxt[PF ? CH : 1];
  float gr[CH][V], br[CH][V];  // this lane's affine parameters, the same for every row it walks
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int i = 0; i < V; i += 4) {
      const int col = (c * 32 + lane) * V + i;
      const float4 g4 = __ldg(reinterpret_cast<const float4*>(gamma + col));
      const float4 b4 = __ldg(reinterpret_cast<const float4*>(beta + col));
      gr[c][i] = g4.x; gr[c][i + 1] = g4.y; gr[c][i + 2] = g4.z; gr[c][i + 3] = g4.w;
      br[c][i] = b4.x; br[c][i + 1] = b4.y; br[c][i + 2] = b4.z; br[c][i + 3] = b4.w;
    }
  float wr[PRED ? CH : 1][V];  // the consumer's checksum vector at this lane's columns (PRED)
  if constexpr (PRED) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
#pragma unroll
      for (int i = 0; i < V; i += 4) {
        const float4 w4 = __ldg(reinterpret_cast<const float4*>(w_pred + (c * 32 + lane) * V + i));
        wr[c][i] = w4.x; wr[c][i + 1] = w4.y; wr[c][i + 2] = w4.z; wr[c][i + 3] = w4.w;
      }
  }
  if (row < rows) {
#pragma unroll
    for (int c = 0; c < CH; ++c) cur[c] = *reinterpret_cast<const uint4*>(h + row * D + (c * 32 + lane) * V);
  }
  for (; row < rows; row += stride) {
    const int64_t nrow = row + stride;
    if constexpr (PF) {
      if (nrow < rows) {
#pragma unroll
        for (int c = 0; c < CH; ++c) nxt[c] = *reinterpret_cast<const uint4*>(h + nrow * D + (c * 32 + lane) * V);
      }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      float v[V];
      Vec<T>::load(&cur[c], v);
#pragma unroll
      for (int i = 0; i < V; ++i) s += v[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mean = s / static_cast<float>(D);
    float q = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      float v[V];
      Vec<T>::load(&cur[c], v);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const float dv = v[i] - mean;
        q += dv * dv;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float rstd = rsqrtf(q / static_cast<float>(D) + eps);
    float p = 0.f;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int col = (c * 32 + lane) * V;
      float v[V], o[V];
      Vec<T>::load(&cur[c], v);
#pragma unroll
      for (int i = 0; i < V; ++i) o[i] = fmaf((v[i] - mean) * rstd, gr[c][i], br[c][i]);
      if constexpr (PRED) {  // add_layernorm_kernel's predicted sum: the same products, the same order
        uint4 packed;
        Vec<T>::store(&packed, o);
        Vec<T>::load(&packed, o);
        *reinterpret_cast<uint4*>(ln_out + row * D + col) = packed;
#pragma unroll
        for (int i = 0; i < V; ++i) p = fmaf(o[i], wr[c][i], p);
      } else {
        Vec<T>::store(ln_out + row * D + col, o);
      }
    }
    if constexpr (PRED) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
      if (lane == 0) pred_out[row] = static_cast<unsigned long long>(__float_as_uint(p));
    }
    if constexpr (PF) {
#pragma unroll
      for (int c = 0; c < CH; ++c) cur[c] = nxt[c];
    } else if (nrow < rows) {
#pragma unroll
      for (int c = 0; c < CH; ++c) cur[c] = *reinterpret_cast<const uint4*>(h + nrow * D + (c * 32 + lane) * V);
    }
  }
}

static int sm_count() {  // of the current device (cached per device)
  static int cached[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cached[dev] == 0) {
    int n = 0;
    cached[dev] = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0 ? n : 148;
  }
  return cached[dev];
}

template <typename T>
int launch_add_ln_t(const void* h, const void* y, int64_t rows, int D, const float* gamma, const float* beta,
                    float eps, void* h_out, void* ln_out, const float* w_pred, unsigned long long* pred_out,
                    cudaStream_t s) {
  constexpr int V = Vec<T>::N;
  if (D % (32 * V) != 0) return fail(GG_EUNSUPPORTED, "add_layernorm: D must be a multiple of 32 x 16 bytes");
  if (ln_out == h || (y != nullptr && ln_out == y) || (h_out != nullptr && ln_out == h_out))
    return fail(GG_EINVAL, "add_layernorm: ln_out must not alias h, y or h_out");
  const int ch = D / (32 * V);
  const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
  const T* hp = static_cast<const T*>(h);
  const T* yp = static_cast<const T*>(y);
  T* ho = static_cast<T*>(h_out);
  T* lo = static_cast<T*>(ln_out);
  if (y == nullptr && (ch == 3 || ch == 4)) {  // ViT-B (768) and ViT-L (1024) widths at 16 bits
    const int64_t want = (rows + 7) / 8;
    const unsigned g = static_cast<unsigned>(std::min<int64_t>(want, static_cast<int64_t>(sm_count()) * GG_LN_STREAM_BPS));
    if (ch == 3) {
      if (w_pred != nullptr)
        layernorm_stream_kernel<T, 3, true><<<g, 256, 0, s>>>(hp, rows, D, gamma, beta, eps, lo, w_pred, pred_out);
      else
        layernorm_stream_kernel<T, 3, false><<<g, 256, 0, s>>>(hp, rows, D, gamma, beta, eps, lo, nullptr, nullptr);
    } else {
      if (w_pred != nullptr)
        layernorm_stream_kernel<T, 4, true><<<g, 256, 0, s>>>(hp, rows, D, gamma, beta, eps, lo, w_pred, pred_out);
      else
        layernorm_stream_kernel<T, 4, false><<<g, 256, 0, s>>>(hp, rows, D, gamma, beta, eps, lo, nullptr, nullptr);
    }
    return check_launch("add_layernorm");
  }
  switch (ch) {
#define GG_LN_CASE(n) \
  case n:                                                                                                    \
    if (w_pred != nullptr)                                                                                   \
      add_layernorm_kernel<T, n, true><<<grid, 256, 0, s>>>(hp, yp, rows, D, gamma, beta, eps, ho, lo, w_pred, \
                                                            pred_out);                                       \
    else                                                                                                     \
      add_layernorm_kernel<T, n, false><<<grid, 256, 0, s>>>(hp, yp, rows, D, gamma, beta, eps, ho, lo, w_pred, \
                                                             pred_out);                                      \
    break;
    GG_LN_CASE(1) GG_LN_CASE(2) GG_LN_CASE(3) GG_LN_CASE(4) GG_LN_CASE(5) GG_LN_CASE(6) GG_LN_CASE(8)
#undef GG_LN_CASE
    default:
      return fail(GG_EUNSUPPORTED, "add_layernorm: row width not built (32 x 16-byte chunks x {1..6, 8})");
  }
  return check_launch("add_layernorm");
}

template <typename T>
int launch_embed_ln_t(const void* e, const void* pos, const void* cls, int64_t B, int T_, int D, const float* gamma,
                      const float* beta, float eps, void* h_out, void* ln_out, const float* w_pred,
                      unsigned long long* pred_out, cudaStream_t s) {
  constexpr int V = Vec<T>::N;
  if (D % (32 * V) != 0) return fail(GG_EUNSUPPORTED, "embed_layernorm: D must be a multiple of 32 x 16 bytes");
  const int ch = D / (32 * V);
  const int64_t rows = B * T_;
  const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
  const T* ep = static_cast<const T*>(e);
  const T* pp = static_cast<const T*>(pos);
  const T* cp = static_cast<const T*>(cls);
  T* ho = static_cast<T*>(h_out);
  T* lo = static_cast<T*>(ln_out);
  switch (ch) {
#define GG_EMB_CASE(n)                                                                                            \
  case n:                                                                                                        \
    if (w_pred != nullptr)                                                                                       \
      add_layernorm_kernel<T, n, true, true><<<grid, 256, 0, s>>>(ep, pp, rows, D, gamma, beta, eps, ho, lo, w_pred, \
                                                                  pred_out, cp, T_);                             \
    else                                                                                                         \
      add_layernorm_kernel<T, n, false, true><<<grid, 256, 0, s>>>(ep, pp, rows, D, gamma, beta, eps, ho, lo,      \
                                                                   w_pred, pred_out, cp, T_);                    \
    break;
    GG_EMB_CASE(1) GG_EMB_CASE(2) GG_EMB_CASE(3) GG_EMB_CASE(4) GG_EMB_CASE(5) GG_EMB_CASE(6) GG_EMB_CASE(8)
#undef GG_EMB_CASE
    default:
      return fail(GG_EUNSUPPORTED, "embed_layernorm: row width not built (32 x 16-byte chunks x {1..6, 8})");
  }
  return check_launch("embed_layernorm");
}

// images [B, C, H, W] -> patches [B * (H/P) * (W/P), C * P * P], row (b, gy, gx), column (c, py, px):
// one thread per 16-byte piece, consecutive threads along the patch row (whole 32 B sectors
// read from each image row, fully coalesced writes)
__global__ void patchify_kernel(const uint4* __restrict__ img, int64_t B, int C, int H, int W, int P, int vec_per_seg,
                                uint4* __restrict__ out) {
  const int Gy = H / P, Gx = W / P;
  const int64_t seg_per_row = static_cast<int64_t>(C) * P;  // (c, py) segments of one patch
  const int64_t total = B * Gy * Gx * seg_per_row * vec_per_seg;
  const int64_t vec_w = static_cast<int64_t>(W) / (P / vec_per_seg);  // 16-byte pieces per image row
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = i % vec_per_seg;
    const int64_t seg = (i / vec_per_seg) % seg_per_row;
    const int64_t row = i / (vec_per_seg * seg_per_row);
    const int64_t c = seg / P, py = seg % P;
    const int64_t b = row / (Gy * Gx), g = row % (Gy * Gx), gy = g / Gx, gx = g % Gx;
    const int64_t src = ((b * C + c) * H + gy * P + py) * vec_w + gx * vec_per_seg + v;
    out[i] = __ldg(img + src);
  }
}

}  // namespace

int launch_patchify(int dtype, const void* images, int64_t B, int64_t C, int64_t H, int64_t W, int64_t P, void* out,
                    cudaStream_t s) {
  const int elem = dtype == GG_F32 ? 4 : (dtype == GG_BF16 || dtype == GG_F16) ? 2 : 0;
  if (elem == 0) return fail(GG_EUNSUPPORTED, "patchify: dtype must be GG_BF16, GG_F16 or GG_F32");
  if (B < 1 || C < 1 || P < 1 || H % P || W % P) return fail(GG_EINVAL, "patchify: H and W must be multiples of P");
  if ((P * elem) % 16 || (reinterpret_cast<uintptr_t>(images) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return fail(GG_EUNSUPPORTED, "patchify: P * element size must be a multiple of 16 bytes, tensors 16-byte aligned");
  const int vec_per_seg = static_cast<int>(P * elem / 16);
  patchify_kernel<<<148 * 16, 256, 0, s>>>(static_cast<const uint4*>(images), B, static_cast<int>(C),
                                          static_cast<int>(H), static_cast<int>(W), static_cast<int>(P), vec_per_seg,
                                          static_cast<uint4*>(out));
  return check_launch("patchify");
}

int launch_embed_layernorm(int dtype, const void* e, const void* pos, const void* cls, int64_t B, int64_t T_,
                           int64_t D, const float* gamma, const float* beta, float eps, void* h_out, void* ln_out,
                           const float* w_pred, unsigned long long* pred_out, cudaStream_t s) {
  if ((w_pred == nullptr) != (pred_out == nullptr)) return fail(GG_EINVAL, "embed_layernorm: w_pred needs pred_out");
  if (B < 1 || T_ < 2 || D < 1) return fail(GG_EINVAL, "embed_layernorm: needs B >= 1, T >= 2 tokens, D >= 1");
  if (e == nullptr || pos == nullptr || cls == nullptr || gamma == nullptr || beta == nullptr || h_out == nullptr ||
      ln_out == nullptr)
    return fail(GG_EINVAL, "embed_layernorm: null argument");
  if ((reinterpret_cast<uintptr_t>(e) | reinterpret_cast<uintptr_t>(pos) | reinterpret_cast<uintptr_t>(cls) |
       reinterpret_cast<uintptr_t>(h_out) | reinterpret_cast<uintptr_t>(ln_out) | reinterpret_cast<uintptr_t>(gamma) |
       reinterpret_cast<uintptr_t>(beta) | reinterpret_cast<uintptr_t>(w_pred)) &
      15)
    return fail(GG_EINVAL, "embed_layernorm: tensors must be 16-byte aligned");
  switch (dtype) {
    case GG_BF16: return launch_embed_ln_t<__nv_bfloat16>(e, pos, cls, B, static_cast<int>(T_), static_cast<int>(D),
                                                          gamma, beta, eps, h_out, ln_out, w_pred, pred_out, s);
    case GG_F16: return launch_embed_ln_t<__half>(e, pos, cls, B, static_cast<int>(T_), static_cast<int>(D), gamma,
                                                  beta, eps, h_out, ln_out, w_pred, pred_out, s);
    case GG_F32: return launch_embed_ln_t<float>(e, pos, cls, B, static_cast<int>(T_), static_cast<int>(D), gamma,
                                                 beta, eps, h_out, ln_out, w_pred, pred_out, s);
    default: return fail(GG_EUNSUPPORTED, "embed_layernorm: dtype must be GG_BF16, GG_F16 or GG_F32");
  }
}

int launch_add_layernorm(int dtype, const void* h, const void* y, int64_t rows, int64_t D, const float* gamma,
                         const float* beta, float eps, void* h_out, void* ln_out, const float* w_pred,
                         unsigned long long* pred_out, cudaStream_t s) {
  if ((w_pred == nullptr) != (pred_out == nullptr)) return fail(GG_EINVAL, "add_layernorm: w_pred needs pred_out");
  if (reinterpret_cast<uintptr_t>(w_pred) & 15) return fail(GG_EINVAL, "add_layernorm: w_pred must be 16-byte aligned");
  if (rows < 1 || D < 1) return fail(GG_EINVAL, "add_layernorm: empty input");
  if (gamma == nullptr || beta == nullptr || ln_out == nullptr) return fail(GG_EINVAL, "add_layernorm: null argument");
  if (y != nullptr && h_out == nullptr) return fail(GG_EINVAL, "add_layernorm: residual update needs h_out");
  if ((reinterpret_cast<uintptr_t>(h) | reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(h_out) |
       reinterpret_cast<uintptr_t>(ln_out) | reinterpret_cast<uintptr_t>(gamma) | reinterpret_cast<uintptr_t>(beta)) &
      15)
    return fail(GG_EINVAL, "add_layernorm: tensors must be 16-byte aligned");
  switch (dtype) {
    case GG_BF16: return launch_add_ln_t<__nv_bfloat16>(h, y, rows, static_cast<int>(D), gamma, beta, eps, h_out, ln_out, w_pred,
                                                       pred_out, s);
    case GG_F16: return launch_add_ln_t<__half>(h, y, rows, static_cast<int>(D), gamma, beta, eps, h_out, ln_out, w_pred,
                                                       pred_out, s);
    case GG_F32: return launch_add_ln_t<float>(h, y, rows, static_cast<int>(D), gamma, beta, eps, h_out, ln_out, w_pred,
                                                       pred_out, s);
    default: return fail(GG_EUNSUPPORTED, "add_layernorm: dtype must be GG_BF16, GG_F16 or GG_F32");
  }
}

}  // namespace gg
