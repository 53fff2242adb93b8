// gg_calib.cu — device calibration statistics and range profiling.
//
//   gg_running_stats  guard.calibrate_epsilon (guard.py:300-355) collects every clean d of
//                     a layer and takes mean and std(ddof=1).  Here each batch of d (the
//                     fused check's output, already on the device) is merged into a
//                     device-resident running (n, mean, M2): Welford within a thread's
//                     contiguous chunk, then Chan's pairwise merge over a fixed tree, so the
//                     result is deterministic and no d ever crosses PCIe.
//   gg_minmax         profiler.profile_ranges (profiler.py:62-80): min / max of a layer's raw
//                     outputs over a dataset, plus its non-finite check (which raises there).
//                     A running (min, max, non-finite count) is updated on the device with
//                     16-byte loads (HBM-bound) and order-independent atomics.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <type_traits>

#include "gg_internal.h"

namespace gg {
namespace {

constexpr int STATS_THREADS = 1024;

struct Moments {
  double n, mean, m2;
};

// Chan et al.: merge (nb, mb, M2b) into (na, ma, M2a).
__device__ __forceinline__ Moments merge(Moments a, Moments b) {
  if (b.n == 0.0) return a;
  if (a.n == 0.0) return b;
  const double n = a.n + b.n;
  const double delta = b.mean - a.mean;
  Moments r;
  r.n = n;
  r.mean = a.mean + delta * (b.n / n);
  r.m2 = a.m2 + b.m2 + delta * delta * (a.n * b.n / n);
  return r;
}

__global__ void __launch_bounds__(STATS_THREADS) running_stats_kernel(const double* d, int64_t n, double* state) {
  __shared__ double s_n[STATS_THREADS], s_mean[STATS_THREADS], s_m2[STATS_THREADS];
  const int t = threadIdx.x;
  const int64_t per = (n + STATS_THREADS - 1) / STATS_THREADS;
  const int64_t i0 = min(n, static_cast<int64_t>(t) * per), i1 = min(n, i0 + per);
  Moments m{0.0, 0.0, 0.0};
  for (int64_t i = i0; i < i1; ++i) {  // Welford over this thread's contiguous chunk
    const double x = d[i];
    m.n += 1.0;
    const double delta = x - m.mean;
    m.mean += delta / m.n;
    m.m2 += delta * (x - m.mean);
  }
  s_n[t] = m.n;
  s_mean[t] = m.mean;
  s_m2[t] = m.m2;
  __syncthreads();
  for (int stride = STATS_THREADS / 2; stride > 0; stride >>= 1) {  // fixed tree: deterministic
    if (t < stride) {
      const Moments r = merge(Moments{s_n[t], s_mean[t], s_m2[t]},
                              Moments{s_n[t + stride], s_mean[t + stride], s_m2[t + stride]});
      s_n[t] = r.n;
      s_mean[t] = r.mean;
      s_m2[t] = r.m2;
    }
    __syncthreads();
  }
  if (t == 0) {
    const Moments r = merge(Moments{state[0], state[1], state[2]}, Moments{s_n[0], s_mean[0], s_m2[0]});
    state[0] = r.n;
    state[1] = r.mean;
    state[2] = r.m2;
  }
}

// Order-preserving map of a double onto uint64 (unsigned comparison == numeric comparison).
__device__ __forceinline__ unsigned long long order_key(double v) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Per-thread running extrema in the output's own arithmetic (exact: min / max never round):
// fp32 for 16/32-bit floats, int32 for int32; one conversion to an order key per thread.
template <int DT>
struct Extrema {
  using V = typename std::conditional<DT == GG_I32, int, float>::type;
  V lo, hi;
  unsigned long long bad;
  __device__ Extrema() : lo(DT == GG_I32 ? V(INT_MAX) : V(INFINITY)), hi(DT == GG_I32 ? V(INT_MIN) : V(-INFINITY)), bad(0) {}
  __device__ __forceinline__ void take(V v) {
    if constexpr (DT == GG_I32) {
      lo = min(lo, v);
      hi = max(hi, v);
    } else {
      if (!isfinite(v)) {
        ++bad;
        return;
      }
      lo = fminf(lo, v);
      hi = fmaxf(hi, v);
    }
  }
  __device__ __forceinline__ void word(uint32_t u) {
    if constexpr (DT == GG_BF16) {
      take(__uint_as_float(u << 16));
      take(__uint_as_float(u & 0xFFFF0000u));
    } else if constexpr (DT == GG_F16) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&u));
      take(f.x);
      take(f.y);
    } else if constexpr (DT == GG_F32) {
      take(__uint_as_float(u));
    } else {
      take(static_cast<int>(u));
    }
  }
  __device__ __forceinline__ void elem(const uint8_t* p) {
    if constexpr (DT == GG_BF16) take(__bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p)));
    else if constexpr (DT == GG_F16) take(__half2float(*reinterpret_cast<const __half*>(p)));
    else if constexpr (DT == GG_F32) take(*reinterpret_cast<const float*>(p));
    else take(*reinterpret_cast<const int*>(p));
  }
};

template <int DT>
__global__ void __launch_bounds__(256) minmax_kernel(const uint8_t* y, int64_t M, int64_t N, int64_t ld_bytes, int elem,
                                                     bool vec, unsigned long long* state) {
  Extrema<DT> ex;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (vec && ld_bytes == N * elem) {  // contiguous rows: one flat stream of 16-byte units
    const uint4* p = reinterpret_cast<const uint4*>(y);
    const int64_t units = M * N * elem / 16;
    int64_t u = tid;
    for (; u + stride < units; u += 2 * stride) {  // two loads in flight per thread
      const uint4 a = __ldcs(p + u), b = __ldcs(p + u + stride);
      ex.word(a.x);
      ex.word(a.y);
      ex.word(a.z);
      ex.word(a.w);
      ex.word(b.x);
      ex.word(b.y);
      ex.word(b.z);
      ex.word(b.w);
    }
    if (u < units) {
      const uint4 a = __ldcs(p + u);
      ex.word(a.x);
      ex.word(a.y);
      ex.word(a.z);
      ex.word(a.w);
    }
  } else if (vec) {  // 16-byte units; every row is a whole number of units
    const int64_t units = N * elem / 16;
    for (int64_t u = tid; u < M * units; u += stride) {
      const int64_t r = u / units, c = u - r * units;
      const uint4 w = __ldcs(reinterpret_cast<const uint4*>(y + r * ld_bytes) + c);
      ex.word(w.x);
      ex.word(w.y);
      ex.word(w.z);
      ex.word(w.w);
    }
  } else {
    for (int64_t e = tid; e < M * N; e += stride) {
      const int64_t r = e / N, c = e - r * N;
      ex.elem(y + r * ld_bytes + c * elem);
    }
  }
  const bool any = ex.lo <= ex.hi;  // false only when this thread saw no finite value
  unsigned long long lo = any ? order_key(static_cast<double>(ex.lo)) : ~0ull;
  unsigned long long hi = any ? order_key(static_cast<double>(ex.hi)) : 0ull;
  unsigned long long bad = ex.bad;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __shared__ unsigned long long s_lo[8], s_hi[8], s_bad[8];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_lo[w] = lo;
    s_hi[w] = hi;
    s_bad[w] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < static_cast<int>(blockDim.x >> 5); ++i) {
      lo = s_lo[i] < lo ? s_lo[i] : lo;
      hi = s_hi[i] > hi ? s_hi[i] : hi;
      bad += s_bad[i];
    }
    if (lo != ~0ull) atomicMin(&state[0], lo);
    if (hi != 0ull) atomicMax(&state[1], hi);
    if (bad) atomicAdd(&state[2], bad);
  }
}

}  // namespace

int launch_running_stats(const double* d, int64_t n, double* state, cudaStream_t s) {
  if (n < 0) return fail(GG_EINVAL, "running_stats: negative length");
  if (state == nullptr || (n > 0 && d == nullptr)) return fail(GG_EINVAL, "running_stats: null pointer");
  if (n == 0) return 0;
  running_stats_kernel<<<1, STATS_THREADS, 0, s>>>(d, n, state);
  return check_launch("running_stats");
}

int launch_minmax(int dtype, const void* Y, int64_t M, int64_t N, int64_t ldy, unsigned long long* state,
                  cudaStream_t s) {
  if (M < 0 || N < 0 || ldy < N) return fail(GG_EINVAL, "minmax: bad shape");
  if (state == nullptr || (M * N > 0 && Y == nullptr)) return fail(GG_EINVAL, "minmax: null pointer");
  int elem;
  switch (dtype) {
    case GG_BF16: case GG_F16: elem = 2; break;
    case GG_F32: case GG_I32: elem = 4; break;
    default: return fail(GG_EUNSUPPORTED, "minmax: dtype must be bf16, f16, f32 or i32 (GEMM outputs)");
  }
  if (M * N == 0) return 0;
  const int64_t ld_bytes = ldy * elem;
  const bool vec = (reinterpret_cast<uintptr_t>(Y) % 16 == 0) && (N * elem) % 16 == 0 && ld_bytes % 16 == 0;
  const int64_t work = vec ? M * N * elem / 16 : M * N;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t want = (work + 255) / 256;
  const unsigned grid = static_cast<unsigned>(want < 8 * sms ? (want > 0 ? want : 1) : 8 * sms);
  const uint8_t* y = static_cast<const uint8_t*>(Y);
  switch (dtype) {
    case GG_BF16: minmax_kernel<GG_BF16><<<grid, 256, 0, s>>>(y, M, N, ld_bytes, elem, vec, state); break;
    case GG_F16: minmax_kernel<GG_F16><<<grid, 256, 0, s>>>(y, M, N, ld_bytes, elem, vec, state); break;
    case GG_F32: minmax_kernel<GG_F32><<<grid, 256, 0, s>>>(y, M, N, ld_bytes, elem, vec, state); break;
    default: minmax_kernel<GG_I32><<<grid, 256, 0, s>>>(y, M, N, ld_bytes, elem, vec, state); break;
  }
  return check_launch("minmax");
}

}  // namespace gg
