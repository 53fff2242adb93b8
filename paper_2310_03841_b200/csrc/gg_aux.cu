// gg_aux.cu — reference-exact kernels of the checksum path (CUDA cores).
//
// These reproduce the reference's NumPy folds bit-for-bit: every reduction
// is an ascending, single-accumulator fold that STARTS FROM THE FIRST ELEMENT
// (np.add.accumulate semantics, numerics.py:211-215, guard.py:135-139), every
// product is rounded in the accumulation type before the add (no FMA
// contraction: __dmul_rn/__dadd_rn, __fmul_rn/__fadd_rn), and binary16
// arithmetic is "compute in binary32, round to binary16" (NumPy's HALF loops).
//
//   K2  offline_checksum_kernel   guard.offline_checksum    guard.py:142-160
//   --  verify_rows_kernel        guard._discrepancies +    guard.py:163-215
//                                 guard._verify_arrays
//   K3  flip_bits_kernel          numerics.flip_bit         numerics.py:308-321
//   --  gemm_exact_kernel         numerics.gemm             numerics.py:222-289
//   --  reduce_kernel             numerics.reduce_rows/cols numerics.py:292-305
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <type_traits>

#include "gg_internal.h"

namespace gg {
namespace {

// ------------------------------------------------------------ element access
__device__ __forceinline__ double load_as_f64(const void* base, int dt, int64_t i) {
  switch (dt) {
    case GG_F64: return static_cast<const double*>(base)[i];
    case GG_F32: return static_cast<double>(static_cast<const float*>(base)[i]);
    case GG_F16: return static_cast<double>(__half2float(static_cast<const __half*>(base)[i]));
    case GG_BF16: return static_cast<double>(__bfloat162float(static_cast<const __nv_bfloat16*>(base)[i]));
    case GG_I8: return static_cast<double>(static_cast<const int8_t*>(base)[i]);
    case GG_I32: return static_cast<double>(static_cast<const int32_t*>(base)[i]);
    case GG_I64: return static_cast<double>(static_cast<const long long*>(base)[i]);
  }
  return 0.0;
}
__device__ __forceinline__ long long load_as_i64(const void* base, int dt, int64_t i) {
  switch (dt) {
    case GG_I8: return static_cast<long long>(static_cast<const int8_t*>(base)[i]);
    case GG_I32: return static_cast<long long>(static_cast<const int32_t*>(base)[i]);
    case GG_I64: return static_cast<const long long*>(base)[i];
  }
  return 0;
}

// "astype(acc)" of a stored element, exactly as NumPy converts it.
// f16: double->half is a single RNE rounding (npy_double_to_half); f32 values
// are exact in double, so float->half via double is the same single rounding.
struct AccF64 {
  using T = double;
  __device__ static T from(const void* b, int dt, int64_t i) { return load_as_f64(b, dt, i); }
  __device__ static T add(T a, T b) { return __dadd_rn(a, b); }
  __device__ static T mul(T a, T b) { return __dmul_rn(a, b); }
  __device__ static T sub(T a, T b) { return __dsub_rn(a, b); }
  __device__ static double to_f64(T a) { return a; }
};
struct AccF32 {
  using T = float;
  __device__ static T from(const void* b, int dt, int64_t i) {
    if (dt == GG_F32) return static_cast<const float*>(b)[i];
    return __double2float_rn(load_as_f64(b, dt, i));
  }
  __device__ static T add(T a, T b) { return __fadd_rn(a, b); }
  __device__ static T mul(T a, T b) { return __fmul_rn(a, b); }
  __device__ static T sub(T a, T b) { return __fsub_rn(a, b); }
  __device__ static double to_f64(T a) { return static_cast<double>(a); }
};
struct AccF16 {  // value held as the float of a half; every result re-rounded to half
  using T = float;
  __device__ static float rnd(float v) { return __half2float(__float2half_rn(v)); }
  __device__ static T from(const void* b, int dt, int64_t i) {
    if (dt == GG_F16) return __half2float(static_cast<const __half*>(b)[i]);
    return __half2float(__double2half(load_as_f64(b, dt, i)));
  }
  __device__ static T add(T a, T b) { return rnd(__fadd_rn(a, b)); }
  __device__ static T mul(T a, T b) { return rnd(__fmul_rn(a, b)); }
  __device__ static T sub(T a, T b) { return rnd(__fsub_rn(a, b)); }
  __device__ static double to_f64(T a) { return static_cast<double>(a); }
};
struct AccI64 {
  using T = long long;
  __device__ static T from(const void* b, int dt, int64_t i) { return load_as_i64(b, dt, i); }
  __device__ static T add(T a, T b) { return static_cast<T>(static_cast<unsigned long long>(a) + static_cast<unsigned long long>(b)); }
  __device__ static T mul(T a, T b) { return static_cast<T>(static_cast<unsigned long long>(a) * static_cast<unsigned long long>(b)); }
  __device__ static T sub(T a, T b) { return static_cast<T>(static_cast<unsigned long long>(a) - static_cast<unsigned long long>(b)); }
  __device__ static double to_f64(T a) { return static_cast<double>(a); }
};

template <class A>
__device__ __forceinline__ void store_acc(void* out, int64_t i, typename A::T v);
template <>
__device__ __forceinline__ void store_acc<AccF64>(void* out, int64_t i, double v) { static_cast<double*>(out)[i] = v; }
template <>
__device__ __forceinline__ void store_acc<AccF32>(void* out, int64_t i, float v) { static_cast<float*>(out)[i] = v; }
template <>
__device__ __forceinline__ void store_acc<AccF16>(void* out, int64_t i, float v) {
  static_cast<__half*>(out)[i] = __float2half_rn(v);
}
template <>
__device__ __forceinline__ void store_acc<AccI64>(void* out, int64_t i, long long v) {
  static_cast<long long*>(out)[i] = v;
}

// ------------------------------------------------------------ K2 offline checksum
// w_sum[k] = fold_n W(k, n); W(k, n) = layout 0: W[n*ldw + k] (torch [N,K]);
// layout 1: Wt[k*ldw + n] (reference [K,N]).
// One thread per k folds n = 0..N-1 in ascending order (bit-exact with the
// reference's fold); the source dtype is a template constant and the loads of 32
// rows are issued ahead of their adds, so the kernel runs at memory-level
// parallelism instead of one dependent load per add.
template <class A, int DT>
__global__ void __launch_bounds__(64) offline_checksum_kernel(const void* W, int64_t K, int64_t N, int64_t ldw,
                                                             int layout, void* w_sum) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= K) return;
  auto idx = [&](int64_t n) { return layout == 0 ? n * ldw + k : k * ldw + n; };
  using T = typename A::T;
  T acc = A::from(W, DT, idx(0));
  constexpr int U = 32;
  int64_t n = 1;
  for (; n + U <= N; n += U) {
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = A::from(W, DT, idx(n + u));
#pragma unroll
    for (int u = 0; u < U; ++u) acc = A::add(acc, v[u]);
  }
  for (; n < N; ++n) acc = A::add(acc, A::from(W, DT, idx(n)));
  store_acc<A>(w_sum, k, acc);
}
template <class A>
int launch_k2(int w_dtype, const void* W, int64_t K, int64_t N, int64_t ldw, int layout, void* w_sum, cudaStream_t s) {
  const unsigned g = static_cast<unsigned>((K + 63) / 64);
  switch (w_dtype) {
#define GG_K2_CASE(DTV)                                                                         \
  case DTV:                                                                                     \
    offline_checksum_kernel<A, DTV><<<g, 64, 0, s>>>(W, K, N, ldw, layout, w_sum);           \
    return 0;
    GG_K2_CASE(GG_F64)
    GG_K2_CASE(GG_F32)
    GG_K2_CASE(GG_F16)
    GG_K2_CASE(GG_BF16)
    GG_K2_CASE(GG_I8)
    GG_K2_CASE(GG_I32)
    GG_K2_CASE(GG_I64)
#undef GG_K2_CASE
  }
  return fail(GG_EINVAL, "offline_checksum: bad weight dtype");
}
// bias_sum = fold_n bias[n] (ascending, one thread; loads issued 32 ahead of the adds)
template <class A, int DT>
__global__ void vector_sum_kernel(const void* v, int64_t n, void* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  using T = typename A::T;
  T acc;
  if (v == nullptr || n == 0) {
    acc = T(0);
  } else {
    acc = A::from(v, DT, 0);
    constexpr int U = 32;
    int64_t i = 1;
    for (; i + U <= n; i += U) {
      T x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = A::from(v, DT, i + u);
#pragma unroll
      for (int u = 0; u < U; ++u) acc = A::add(acc, x[u]);
    }
    for (; i < n; ++i) acc = A::add(acc, A::from(v, DT, i));
  }
  store_acc<A>(out, 0, acc);
}
template <class A>
void launch_vector_sum(int dtype, const void* v, int64_t n, void* out, cudaStream_t s) {
  switch (dtype) {
#define GG_VS_CASE(DTV)                                            \
  case DTV:                                                        \
    vector_sum_kernel<A, DTV><<<1, 32, 0, s>>>(v, n, out);         \
    return;
    GG_VS_CASE(GG_F64)
    GG_VS_CASE(GG_F32)
    GG_VS_CASE(GG_F16)
    GG_VS_CASE(GG_BF16)
    GG_VS_CASE(GG_I8)
    GG_VS_CASE(GG_I32)
    GG_VS_CASE(GG_I64)
#undef GG_VS_CASE
  }
  vector_sum_kernel<A, GG_F64><<<1, 32, 0, s>>>(nullptr, 0, out);  // no bias: sum 0
}

// ------------------------------------------------------------ verify (exact)
__device__ __forceinline__ unsigned long long gap_key(double gap) {
  if (gap != gap) return 0ull;
  return static_cast<unsigned long long>(__double_as_longlong(gap)) + 1ull;
}

template <class A>
__device__ __forceinline__ typename A::T load_wsum(const void* w_sum, int64_t k) {
  if constexpr (std::is_same<A, AccI64>::value) return static_cast<const long long*>(w_sum)[k];
  else if constexpr (std::is_same<A, AccF64>::value) return static_cast<const double*>(w_sum)[k];
  else if constexpr (std::is_same<A, AccF32>::value) return static_cast<const float*>(w_sum)[k];
  else return __half2float(static_cast<const __half*>(w_sum)[k]);
}

// One thread per row: the two folds of guard._discrepancies in the checksum
// precision, then the flag rule of guard._verify_arrays.
template <class A>
__global__ void verify_rows_kernel(int x_dtype, const void* X, int64_t M, int64_t K, int64_t ldx, int y_dtype,
                                   const void* Y, int64_t N, int64_t ldy, const void* w_sum, const void* bias_sum,
                                   double lo, double hi, void* d_out, uint8_t* flags) {
  const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (b >= M) return;
  using T = typename A::T;
  // predicted = fold_k(x[b,k] * w_sum[k]) + bias_sum      (guard.py:168-169)
  T pred = A::mul(A::from(X, x_dtype, b * ldx + 0), load_wsum<A>(w_sum, 0));
  for (int64_t k = 1; k < K; ++k) pred = A::add(pred, A::mul(A::from(X, x_dtype, b * ldx + k), load_wsum<A>(w_sum, k)));
  pred = A::add(pred, load_wsum<A>(bias_sum, 0));
  // observed = fold_n(y[b,n])                              (guard.py:170)
  T obs = A::from(Y, y_dtype, b * ldy + 0);
  for (int64_t n = 1; n < N; ++n) obs = A::add(obs, A::from(Y, y_dtype, b * ldy + n));
  const T dd = A::sub(pred, obs);
  bool flag;
  if constexpr (std::is_same<A, AccI64>::value) {
    static_cast<long long*>(d_out)[b] = dd;
    flag = dd != 0;  // guard.py:193
  } else {
    const double d = A::to_f64(dd);
    static_cast<double*>(d_out)[b] = d;
    flag = !((d >= lo) && (d <= hi));  // guard.py:204
  }
  flags[b] = flag ? 1 : 0;
}

// NumPy's pairwise summation (np.add.reduce on a contiguous float64 array),
// iterative form of pairwise_sum in numpy/_core/src/umath/loops_utils.h.src.
// Leaf of the recursion (n <= 128): unrolled by 8, as NumPy.
__device__ double np_pairwise_leaf(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  return 0.0;  // unreachable: callers pass n <= 128
}

__device__ double np_pairwise_sum(const double* a, int64_t n) {
  if (n <= 128) return np_pairwise_leaf(a, n);
  // explicit stack of (offset, length, partial-left-result state)
  struct Frame { int64_t off, len; int state; double left; };
  Frame st[64];
  int sp = 0;
  st[0] = {0, n, 0, 0.0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame& f = st[sp];
    if (f.len <= 128) {
      ret = np_pairwise_leaf(a + f.off, f.len);
      --sp;
      continue;
    }
    int64_t n2 = f.len / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st[sp + 1] = {f.off, n2, 0, 0.0};
      ++sp;
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[sp + 1] = {f.off + n2, f.len - n2, 0, 0.0};
      ++sp;
    } else {
      ret = __dadd_rn(f.left, ret);
      --sp;
    }
  }
  return ret;
}

// The same sum computed by one block: the recursion's leaves (<= 128 contiguous
// elements, split points fixed by n alone) are summed by separate threads with
// the leaf routine above, then thread 0 combines them in the recursion's order,
// so the result is bit-identical to the serial form.  Falls back to the serial
// walk when n has more leaves than fit in shared memory.
constexpr int PW_MAX_LEAVES = 2048;
__device__ double np_pairwise_sum_block(const double* a, int64_t n) {
  __shared__ long long s_leaf[PW_MAX_LEAVES];  // off << 8 | len
  __shared__ double s_val[PW_MAX_LEAVES];
  __shared__ int s_nleaf;
  __shared__ double s_res;
  if (threadIdx.x == 0) {
    // pre-order walk listing the leaves left to right
    int64_t st_off[64], st_len[64];
    int sp = 0, nl = 0;
    st_off[0] = 0;
    st_len[0] = n;
    while (sp >= 0 && nl <= PW_MAX_LEAVES) {
      const int64_t off = st_off[sp], len = st_len[sp];
      --sp;
      if (len <= 128) {
        if (nl < PW_MAX_LEAVES) s_leaf[nl] = (static_cast<long long>(off) << 8) | len;
        ++nl;
        continue;
      }
      int64_t n2 = len / 2;
      n2 -= n2 % 8;
      st_off[++sp] = off + n2;  // right child popped after the left one
      st_len[sp] = len - n2;
      st_off[++sp] = off;
      st_len[sp] = n2;
    }
    s_nleaf = nl;
  }
  __syncthreads();
  const int nl = s_nleaf;
  if (nl > PW_MAX_LEAVES) {
    if (threadIdx.x == 0) s_res = np_pairwise_sum(a, n);
    __syncthreads();
    return s_res;
  }
  for (int i = threadIdx.x; i < nl; i += blockDim.x)
    s_val[i] = np_pairwise_leaf(a + (s_leaf[i] >> 8), s_leaf[i] & 0xff);
  __syncthreads();
  if (threadIdx.x == 0) {
    // post-order combine: the same tree, leaves consumed in order
    struct Fr { int64_t len; int state; double left; };
    Fr st[64];
    int sp = 0, li = 0;
    st[0] = {n, 0, 0.0};
    double ret = 0.0;
    while (sp >= 0) {
      Fr& f = st[sp];
      if (f.len <= 128) {
        ret = s_val[li++];
        --sp;
        continue;
      }
      int64_t n2 = f.len / 2;
      n2 -= n2 % 8;
      if (f.state == 0) {
        f.state = 1;
        st[sp + 1] = {n2, 0, 0.0};
        ++sp;
      } else if (f.state == 1) {
        f.left = ret;
        f.state = 2;
        st[sp + 1] = {f.len - n2, 0, 0.0};
        ++sp;
      } else {
        ret = __dadd_rn(f.left, ret);
        --sp;
      }
    }
    s_res = ret;
  }
  __syncthreads();
  return s_res;
}

// One block: launch summaries of guard._verify_arrays over all rows
// (deterministic: integer sum / max of order-preserving keys).
__global__ void verify_finish_kernel(int64_t M, bool is_int, int statistic, double mu, double lo, double hi,
                                     const void* d, uint8_t* flags, double* max_disc, int* nflag,
                                     uint8_t* triggered) {
  __shared__ int s_n[32];
  __shared__ unsigned long long s_k[32];
  __shared__ int s_batch_flag;
  if (!is_int && statistic == GG_BATCH_MEAN) {
    // dm = float(d.mean()) = pairwise_sum(d) / n               (guard.py:199-201)
    const double dm = __ddiv_rn(np_pairwise_sum_block(static_cast<const double*>(d), M), static_cast<double>(M));
    if (threadIdx.x == 0) s_batch_flag = ((lo <= dm) && (dm <= hi)) ? 0 : 1;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < M; i += blockDim.x) flags[i] = static_cast<uint8_t>(s_batch_flag);
  }
  int nf = 0;
  unsigned long long key = 0;
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
    if (is_int) {
      const long long v = static_cast<const long long*>(d)[i];
      const unsigned long long mag = v < 0 ? 0ull - static_cast<unsigned long long>(v) : static_cast<unsigned long long>(v);
      const unsigned long long k = gap_key(static_cast<double>(mag));  // float(np.abs(d).max())
      key = k > key ? k : key;
      nf += v != 0 ? 1 : 0;
    } else {
      const unsigned long long k = gap_key(fabs(static_cast<const double*>(d)[i] - mu));  // guard.py:205-207
      key = k > key ? k : key;
      nf += (statistic == GG_BATCH_MEAN) ? s_batch_flag : flags[i];
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    nf += __shfl_xor_sync(0xffffffffu, nf, o);
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, key, o);
    key = w > key ? w : key;
  }
  if ((threadIdx.x & 31) == 0) { s_n[threadIdx.x >> 5] = nf; s_k[threadIdx.x >> 5] = key; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int tn = 0;
    unsigned long long tk = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { tn += s_n[w]; tk = s_k[w] > tk ? s_k[w] : tk; }
    *max_disc = (tk == 0ull) ? __longlong_as_double(0x7FF0000000000000ll) : __longlong_as_double(static_cast<long long>(tk - 1ull));
    *nflag = tn;
    *triggered = tn > 0 ? 1 : 0;
  }
}

// ------------------------------------------------------------ K3 flips
__global__ void flip_bits_kernel(uint8_t* base, int elem_bytes, const int64_t* elem_idx, const int32_t* bit_idx,
                                 int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int64_t e = elem_idx[i];
  const int bit = bit_idx[i];
  // bit b of a little-endian element lives in byte b/8 at position b%8
  uint8_t* byte = base + e * elem_bytes + (bit >> 3);
  // serial per element: atomics keep two flips of one byte from racing
  const uintptr_t addr = reinterpret_cast<uintptr_t>(byte);
  unsigned int* word = reinterpret_cast<unsigned int*>(addr & ~uintptr_t(3));
  const unsigned int shift = static_cast<unsigned int>((addr & 3u) * 8u + (bit & 7));
  atomicXor(word, 1u << shift);
}

// ------------------------------------------------------------ exact GEMM
// Y[b,o] = fold_k(x[b,k]*w[k,o]) (+ bias[o]) in the accumulation type, then
// rounded to the operand dtype.  numerics._gemm_accumulate starts the fold at
// the first product when B*I*O <= 2^26 (np.add.accumulate) and at zero
// otherwise (the k-loop path); both are reproduced (start_zero).
template <class A>
__global__ void gemm_exact_kernel(int dtype, const void* X, int64_t M, int64_t K, const void* Wt, int64_t N,
                                  const void* bias, void* Y, bool start_zero) {
  const int64_t o = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (o >= N) return;
  using T = typename A::T;
  for (int64_t b = blockIdx.y; b < M; b += gridDim.y) {
    T acc;
    int64_t k0;
    if (start_zero) {
      acc = T(0);
      k0 = 0;
    } else {
      acc = A::mul(A::from(X, dtype, b * K), A::from(Wt, dtype, o));
      k0 = 1;
    }
    for (int64_t k = k0; k < K; ++k)
      acc = A::add(acc, A::mul(A::from(X, dtype, b * K + k), A::from(Wt, dtype, k * N + o)));
    if (bias) acc = A::add(acc, A::from(bias, GG_F64, o));  // bias.astype(acc)
    const double v = A::to_f64(acc);
    if (dtype == GG_F64) static_cast<double*>(Y)[b * N + o] = v;
    else if (dtype == GG_F32) static_cast<float*>(Y)[b * N + o] = __double2float_rn(v);
    else if (dtype == GG_F16) static_cast<__half*>(Y)[b * N + o] = __double2half(v);
    else static_cast<__nv_bfloat16*>(Y)[b * N + o] = __double2bfloat16(v);
  }
}
// int32 accumulation for integer operands: products and sums wrap in int32
// (X.astype(int32) * Wt.astype(int32), numerics.py:267-272).
struct AccI32 {
  using T = int;
  __device__ static T add(T a, T b) { return static_cast<T>(static_cast<unsigned>(a) + static_cast<unsigned>(b)); }
  __device__ static T mul(T a, T b) { return static_cast<T>(static_cast<unsigned>(a) * static_cast<unsigned>(b)); }
};
template <typename E>
__global__ void gemm_exact_int_kernel(const E* x, int64_t M, int64_t K, const E* w, int64_t N, const int32_t* bias,
                                      int32_t* Y, bool start_zero) {
  const int64_t o = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (o >= N) return;
  for (int64_t b = blockIdx.y; b < M; b += gridDim.y) {
    int acc;
    int64_t k0;
    if (start_zero) { acc = 0; k0 = 0; }
    else { acc = AccI32::mul(static_cast<int>(x[b * K]), static_cast<int>(w[o])); k0 = 1; }
    for (int64_t k = k0; k < K; ++k)
      acc = AccI32::add(acc, AccI32::mul(static_cast<int>(x[b * K + k]), static_cast<int>(w[k * N + o])));
    if (bias) acc = AccI32::add(acc, bias[o]);
    Y[b * N + o] = acc;
  }
}

// ------------------------------------------------------------ reductions
__global__ void reduce_kernel(int dtype, const void* A, int64_t rows, int64_t cols, int axis, void* out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool is_int = (dtype == GG_I8 || dtype == GG_I32 || dtype == GG_I64);
  const int64_t n_out = axis == 1 ? rows : cols;
  const int64_t len = axis == 1 ? cols : rows;
  if (i >= n_out) return;
  auto idx = [&](int64_t j) { return axis == 1 ? i * cols + j : j * cols + i; };
  if (is_int) {
    long long acc = load_as_i64(A, dtype, idx(0));
    for (int64_t j = 1; j < len; ++j) acc = AccI64::add(acc, load_as_i64(A, dtype, idx(j)));
    static_cast<long long*>(out)[i] = acc;
  } else {
    double acc = load_as_f64(A, dtype, idx(0));
    for (int64_t j = 1; j < len; ++j) acc = __dadd_rn(acc, load_as_f64(A, dtype, idx(j)));
    static_cast<double*>(out)[i] = acc;
  }
}

__global__ void round_kernel(int dtype, const double* in, void* out, int64_t n) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double v = in[i];
  if (dtype == GG_F32) static_cast<float*>(out)[i] = __double2float_rn(v);
  else if (dtype == GG_F16) static_cast<__half*>(out)[i] = __double2half(v);
  else if (dtype == GG_BF16) static_cast<__nv_bfloat16*>(out)[i] = __double2bfloat16(v);
  else static_cast<double*>(out)[i] = v;
}

// w_sum side-path encodings for the fused checksum (see gg_checksum_aux).
// Every encoding is zero-padded to a multiple of 128 K-elements so the GEMM's
// checksum warps read whole K-blocks without bounds checks.
constexpr int64_t AUX_PAD = 128;
inline int64_t aux_padded(int64_t K) { return (K + AUX_PAD - 1) / AUX_PAD * AUX_PAD; }

__global__ void f32_of_f64_kernel(const double* w, int64_t K, int64_t Kp, float* out) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= Kp) return;
  out[k] = k < K ? __double2float_rn(w[k]) : 0.f;
}
__global__ void digits_i64_kernel(const long long* w, int64_t K, int64_t Kp, int4* out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;  // group of 4 k
  if (i * 4 >= Kp) return;
  uint32_t plane[3] = {0u, 0u, 0u};
  for (int e = 0; e < 4; ++e) {
    const int64_t k = i * 4 + e;
    long long v = k < K ? w[k] : 0;
    for (int d = 0; d < 3; ++d) {
      const long long dig = ((v + 128) & 255) - 128;  // signed digit in [-128, 127]
      plane[d] |= (static_cast<uint32_t>(dig) & 0xFFu) << (8 * e);
      v = (v - dig) / 256;
    }
  }
  out[i] = make_int4(static_cast<int>(plane[0]), static_cast<int>(plane[1]), static_cast<int>(plane[2]), 0);
}

// fp32 -> tf32 (10-bit mantissa) rounded to nearest even; non-finite values pass through.
__device__ __forceinline__ float tf32_rne(float x) {
  const uint32_t u = __float_as_uint(x);
  if ((u & 0x7f800000u) == 0x7f800000u) return x;
  const uint32_t r = (u + 0xfffu + ((u >> 13) & 1u)) & 0xffffe000u;
  // rounding up past the largest finite tf32 would give inf: truncate instead
  return ((r & 0x7f800000u) == 0x7f800000u) ? __uint_as_float(u & 0xffffe000u) : __uint_as_float(r);
}

// 3xTF32 expansion of an fp32 operand [rows, K] into [rows, 3 * Ks]:
// role 0 (A / X): [hi | lo | hi], role 1 (B / W): [lo | hi | hi]; hi = tf32(x),
// lo = x - hi (exact in fp32).  The small cross terms come first: the tensor
// core's fp32 accumulator truncates on every step by a fraction of its own
// magnitude, so terms added while it is still small lose almost nothing
// (measured on cfg1: row-sum error 7.7e-5 against 3.5e-4 with hi*hi first).
// A non-finite x is placed whole in the last segment with zeros in the other
// two, so no inf * 0 term appears on either side.
__global__ void split_tf32x3_kernel(const float* __restrict__ src, int64_t rows, int64_t K, int64_t ld, int role,
                                    float* __restrict__ dst, int64_t ldd, int64_t Ks) {
  const int64_t r = blockIdx.y;
  const float* s = src + r * ld;
  float* d = dst + r * ldd;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < Ks;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float h = 0.f, l = 0.f, x = 0.f;
    if (k < K) {
      x = s[k];
      if (isfinite(x)) {
        h = tf32_rne(x);
        l = x - h;
      } else {
        h = x;
      }
    }
    const bool fin = isfinite(x);
    d[k] = fin ? (role == 0 ? h : l) : 0.f;
    d[Ks + k] = fin ? (role == 0 ? l : h) : 0.f;
    d[2 * Ks + k] = h;
  }
}

// checksum side path of a 3xTF32 launch: [0 | w | w] over the three K segments of
// the expanded X [hi | lo | hi] (x = lo + hi enters the predicted sum exactly once)
__global__ void f32x3_of_f64_kernel(const double* w, int64_t K, int64_t Ks, int64_t total, float* out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= total) return;
  const int64_t seg = i / Ks, k = i - seg * Ks;
  out[i] = (seg >= 1 && seg < 3 && k < K) ? __double2float_rn(w[k]) : 0.f;
}

inline unsigned grid1(int64_t n, int bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

}  // namespace

// ====================================================================== launchers
int launch_offline_checksum(int w_dtype, const void* W, int64_t K, int64_t N, int64_t ldw, int w_layout,
                            const void* bias, int bias_dtype, int chk_prec, void* w_sum_out, void* bias_sum_out,
                            cudaStream_t s) {
  const bool w_int = (w_dtype == GG_I8 || w_dtype == GG_I32 || w_dtype == GG_I64);
  // guard.py:148-152
  if (w_int && chk_prec != GG_P_I64) return fail(GG_EINVAL, "integer layers require the int64-exact checksum precision");
  if (!w_int && chk_prec == GG_P_I64) return fail(GG_EINVAL, "int64-exact checksums only apply to integer layers");
  if (K < 1 || N < 1) return fail(GG_EINVAL, "offline_checksum: empty weight");
  if (dtype_bytes(w_dtype) == 0) return fail(GG_EINVAL, "offline_checksum: bad weight dtype");
  switch (chk_prec) {
    case GG_P_F64:
      if (int rc = launch_k2<AccF64>(w_dtype, W, K, N, ldw, w_layout, w_sum_out, s)) return rc;
      launch_vector_sum<AccF64>(bias_dtype, bias, N, bias_sum_out, s);
      break;
    case GG_P_F32:
      if (int rc = launch_k2<AccF32>(w_dtype, W, K, N, ldw, w_layout, w_sum_out, s)) return rc;
      launch_vector_sum<AccF32>(bias_dtype, bias, N, bias_sum_out, s);
      break;
    case GG_P_F16:
      if (int rc = launch_k2<AccF16>(w_dtype, W, K, N, ldw, w_layout, w_sum_out, s)) return rc;
      launch_vector_sum<AccF16>(bias_dtype, bias, N, bias_sum_out, s);
      break;
    case GG_P_I64:
      if (int rc = launch_k2<AccI64>(w_dtype, W, K, N, ldw, w_layout, w_sum_out, s)) return rc;
      launch_vector_sum<AccI64>(bias_dtype, bias, N, bias_sum_out, s);
      break;
    default:
      return fail(GG_EINVAL, "offline_checksum: unknown precision");
  }
  return check_launch("offline_checksum");
}

int launch_verify_rows(int x_dtype, const void* X, int64_t M, int64_t K, int64_t ldx, int y_dtype, const void* Y,
                       int64_t N, int64_t ldy, int chk_prec, const void* w_sum, const void* bias_sum, double mu,
                       double lo, double hi, int statistic, void* d_out, uint8_t* flags_out, double* max_disc_out,
                       int32_t* nflag_out, uint8_t* triggered_out, cudaStream_t s) {
  if (M < 1 || K < 1 || N < 1) return fail(GG_EINVAL, "verify_rows: empty operand");
  if (dtype_bytes(x_dtype) == 0 || dtype_bytes(y_dtype) == 0) return fail(GG_EINVAL, "verify_rows: bad dtype");
  const bool is_int = chk_prec == GG_P_I64;
  const unsigned g = grid1(M, 128);
  switch (chk_prec) {
    case GG_P_F64:
      verify_rows_kernel<AccF64><<<g, 128, 0, s>>>(x_dtype, X, M, K, ldx, y_dtype, Y, N, ldy, w_sum, bias_sum, lo, hi,
                                                   d_out, flags_out);
      break;
    case GG_P_F32:
      verify_rows_kernel<AccF32><<<g, 128, 0, s>>>(x_dtype, X, M, K, ldx, y_dtype, Y, N, ldy, w_sum, bias_sum, lo, hi,
                                                   d_out, flags_out);
      break;
    case GG_P_F16:
      verify_rows_kernel<AccF16><<<g, 128, 0, s>>>(x_dtype, X, M, K, ldx, y_dtype, Y, N, ldy, w_sum, bias_sum, lo, hi,
                                                   d_out, flags_out);
      break;
    case GG_P_I64:
      verify_rows_kernel<AccI64><<<g, 128, 0, s>>>(x_dtype, X, M, K, ldx, y_dtype, Y, N, ldy, w_sum, bias_sum, lo, hi,
                                                   d_out, flags_out);
      break;
    default:
      return fail(GG_EINVAL, "verify_rows: unknown precision");
  }
  verify_finish_kernel<<<1, 256, 0, s>>>(M, is_int, statistic, mu, lo, hi, d_out, flags_out, max_disc_out, nflag_out,
                                         triggered_out);
  return check_launch("verify_rows");
}

int launch_flip_bits(void* ptr, int elem_bytes, const int64_t* elem_idx, const int32_t* bit_idx, int64_t n,
                     cudaStream_t s) {
  if (!(elem_bytes == 1 || elem_bytes == 2 || elem_bytes == 4 || elem_bytes == 8))
    return fail(GG_EINVAL, "flip_bits: element width must be 1, 2, 4 or 8 bytes");
  if (n <= 0) return 0;
  flip_bits_kernel<<<grid1(n, 128), 128, 0, s>>>(static_cast<uint8_t*>(ptr), elem_bytes, elem_idx, bit_idx, n);
  return check_launch("flip_bits");
}

int launch_gemm_exact(int dtype, int accum, const void* X, int64_t M, int64_t K, const void* Wt, int64_t N,
                      const void* bias, void* Y, cudaStream_t s) {
  if (M < 1 || K < 1 || N < 1) return fail(GG_EINVAL, "gemm dims mismatch: empty operand");
  const bool start_zero = (M * K * N) > (int64_t(1) << 26);  // numerics.py:219,225
  dim3 grid(grid1(N, 128), static_cast<unsigned>(M < 65535 ? M : 65535));
  if (dtype == GG_I8 || dtype == GG_I32) {
    if (accum != GG_P_I64) return fail(GG_EINVAL, "integer gemm requires the int64-exact accumulation tag");
    if (dtype == GG_I8)
      gemm_exact_int_kernel<int8_t><<<grid, 128, 0, s>>>(static_cast<const int8_t*>(X), M, K,
                                                         static_cast<const int8_t*>(Wt), N,
                                                         static_cast<const int32_t*>(bias), static_cast<int32_t*>(Y),
                                                         start_zero);
    else
      gemm_exact_int_kernel<int32_t><<<grid, 128, 0, s>>>(static_cast<const int32_t*>(X), M, K,
                                                          static_cast<const int32_t*>(Wt), N,
                                                          static_cast<const int32_t*>(bias),
                                                          static_cast<int32_t*>(Y), start_zero);
    return check_launch("gemm_exact");
  }
  if (dtype != GG_F64 && dtype != GG_F32 && dtype != GG_F16 && dtype != GG_BF16)
    return fail(GG_EINVAL, "gemm_exact: unsupported operand dtype");
  if (accum == GG_P_I64) return fail(GG_EINVAL, "float gemm requires a floating accumulation precision");
  const int width = dtype == GG_F64 ? 64 : dtype == GG_F32 ? 32 : 16;
  const int awidth = accum == GG_P_F64 ? 64 : accum == GG_P_F32 ? 32 : 16;
  if (awidth < width) return fail(GG_EINVAL, "accumulation narrower than operand dtype");
  if (dtype == GG_F16 && awidth < 32) return fail(GG_EINVAL, "binary16-emulated gemm accumulates in binary32 or wider");
  if (accum == GG_P_F64)
    gemm_exact_kernel<AccF64><<<grid, 128, 0, s>>>(dtype, X, M, K, Wt, N, bias, Y, start_zero);
  else
    gemm_exact_kernel<AccF32><<<grid, 128, 0, s>>>(dtype, X, M, K, Wt, N, bias, Y, start_zero);
  return check_launch("gemm_exact");
}

int64_t tf32x3_segment(int64_t K) { return (K + 31) / 32 * 32; }

int launch_split_tf32x3(const float* src, int64_t rows, int64_t K, int64_t ld, int role, float* dst, int64_t ldd,
                        cudaStream_t s) {
  if (rows < 1 || K < 1) return fail(GG_EINVAL, "split_tf32x3: empty operand");
  if (role != 0 && role != 1) return fail(GG_EINVAL, "split_tf32x3: role must be 0 (A) or 1 (B)");
  const int64_t Ks = tf32x3_segment(K);
  if (ld < K || ldd < 3 * Ks) return fail(GG_EINVAL, "split_tf32x3: leading dims too small");
  if (rows > 65535 * 1024) return fail(GG_EINVAL, "split_tf32x3: too many rows");
  const int bs = 256;
  const unsigned gx = static_cast<unsigned>(std::min<int64_t>((Ks + bs - 1) / bs, 64));
  int64_t done = 0;
  while (done < rows) {  // grid.y is limited to 65535 rows per launch
    const int64_t n = std::min<int64_t>(rows - done, 65535);
    split_tf32x3_kernel<<<dim3(gx, static_cast<unsigned>(n)), bs, 0, s>>>(src + done * ld, n, K, ld, role,
                                                                        dst + done * ldd, ldd, Ks);
    done += n;
  }
  return check_launch("split_tf32x3");
}

size_t checksum_aux_bytes(int ab_kind, int64_t K) {
  if (K < 1) return 0;
  const int64_t Kp = aux_padded(K);
  switch (ab_kind) {
    case GG_TF32X3: return static_cast<size_t>(aux_padded(3 * tf32x3_segment(K))) * 4;
    case GG_BF16: case GG_F16: case GG_F32: return static_cast<size_t>(Kp) * 4;
    case GG_I8: return static_cast<size_t>(Kp / 4) * 16;
    default: return 0;
  }
}

int launch_checksum_aux(int ab_kind, const void* w_sum, int64_t K, void* aux, cudaStream_t s) {
  if (K < 1) return fail(GG_EINVAL, "checksum_aux: empty w_sum");
  const int64_t Kp = aux_padded(K);
  switch (ab_kind) {
    case GG_TF32X3: {
      const int64_t Ks = tf32x3_segment(K), total = aux_padded(3 * Ks);
      f32x3_of_f64_kernel<<<grid1(total, 256), 256, 0, s>>>(static_cast<const double*>(w_sum), K, Ks, total,
                                                             static_cast<float*>(aux));
      break;
    }
    case GG_BF16: case GG_F16: case GG_F32:
      f32_of_f64_kernel<<<grid1(Kp, 256), 256, 0, s>>>(static_cast<const double*>(w_sum), K, Kp,
                                                       static_cast<float*>(aux));
      break;
    case GG_I8:
      digits_i64_kernel<<<grid1(Kp / 4, 256), 256, 0, s>>>(static_cast<const long long*>(w_sum), K, Kp,
                                                           static_cast<int4*>(aux));
      break;
    default:
      return fail(GG_EINVAL, "checksum_aux: unknown ab_kind");
  }
  return check_launch("checksum_aux");
}

int launch_batch_mean_finish(int64_t M, double mu, double lo, double hi, const double* d, uint8_t* flags,
                             double* max_disc, int32_t* nflag, uint8_t* triggered, cudaStream_t s) {
  verify_finish_kernel<<<1, 256, 0, s>>>(M, false, GG_BATCH_MEAN, mu, lo, hi, d, flags, max_disc, nflag, triggered);
  return check_launch("batch_mean_finish");
}

int launch_reduce(int dtype, const void* A, int64_t rows, int64_t cols, int axis, void* out, cudaStream_t s) {
  if (rows < 1 || cols < 1) return fail(GG_EINVAL, "reduce of empty matrix");
  const int64_t n = axis == 1 ? rows : cols;
  reduce_kernel<<<grid1(n, 128), 128, 0, s>>>(dtype, A, rows, cols, axis, out);
  return check_launch("reduce");
}

int launch_round(int dtype, const double* in, void* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return 0;
  round_kernel<<<grid1(n, 256), 256, 0, s>>>(dtype, in, out, n);
  return check_launch("round");
}

}  // namespace gg
