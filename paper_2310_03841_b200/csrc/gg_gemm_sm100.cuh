// gg_gemm_sm100.cuh — shared definitions of the protected GEMM (K1/K4):
// operand / output kinds, launch parameters, workspace, epilogue conversions.
// The kernel itself is the CTA-pair kernel in gg_gemm2_sm100.cuh.
//
//   C[m, n] = sum_k A[m, k] * B[n, k] + bias[n]
//   d[m]    = (sum_k A[m, k] * w_sum[k] + bias_sum) - sum_n C[m, n]
//   flags   = guard._verify_arrays rule on d            (guard.py:188-215)
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "gg_sm100.cuh"
#include "../../include/gemmguard_b200.h"

namespace gg {

constexpr int BM = 128;  // rows of one checksum band (one CTA of a pair)
constexpr int BN = 256;  // N of one tile

// operand kinds (template KIND)
enum : int { K_BF16 = 0, K_F16 = 1, K_TF32 = 2, K_I8 = 3 };
// output kinds (template OUT)
enum : int { O_BF16 = 0, O_F16 = 1, O_F32 = 2, O_I32 = 3, O_I8 = 4 /* int32 GEMM output, stored requantised */ };

struct Workspace {
  unsigned long long* summary;  // [2] {done bands << 32 | flagged rows, max gap key}: one 128-bit CAS per band
  int* counters;        // [1] active 128-row bands, [2] active 256-row band pairs (replay), [3] tiny-launch tiles
  int* active_pairs;    // [m_pairs] replay: ascending list of the band pairs to recompute
  int* band_counter;    // [m_tiles]
  uint8_t* band_active; // [m_tiles]
  int* band_nflag;      // [m_tiles]
  unsigned long long* band_maxkey;  // [m_tiles]
  double* pred;         // [n_tiles * m_pad] predicted partials (i64 bits for int)
  double* partial;      // [n_tiles * m_pad] observed partials (i64 bits for int)
};

struct Params {
  int M, N, K;
  int m_tiles, n_tiles, k_blocks, m_pad;
  const void* A;        // X [M, K] (read by the checksum warps)
  long long lda;
  void* C;
  long long ldc;
  const void* bias;
  // checksum
  const void* w_sum;    // f64 or i64
  const void* w_aux;    // gg_checksum_aux encoding (bf16/f16: f32, tf32: f64, i8: int32x4 digit planes)
  int w_aux_bytes;      // its padded size
  double bias_sum_f;
  long long bias_sum_i;
  double mu, lo, hi;
  // the same, prepared on the host for the FP64-free band finish: bias_sum_f and -mu as
  // fp32 (hi, lo) pairs (hi in the low word), lo / hi as binary64 order keys
  unsigned long long bias_df, neg_mu_df, lo_key, hi_key;
  int mu_zero;          // mu == 0: the gap is |d|
  int statistic;
  void* d;
  uint8_t* flags;
  double* max_disc;
  int* nflag;
  uint8_t* triggered;
  const gg_injection* inj;
  int n_inj;
  int c_tma;            // 1: C is stored through smem boxes + TMA (needs 16 B aligned C and pitch)
  int sched;            // 0: contiguous tile range per pair, 1: strided (long K)
  int tiny;             // <= 1 tile per pair, <= 4 bands: one launch-wide fold from smem (fewest round trips)
  int few_tiles;        // <= 2 tiles per pair: a split band is folded at the kernel end by all threads of the CTA completing it
  int dbg;              // diagnostics only ($GG_DEBUG), 0 in production: 1 skip predicted dot products,
                        // 2 decouple the checksum warps from the stages, 4 skip band folds, 8 skip
                        // observed sums, 16 relaxed (unordered) split-band counts, 32 drop the
                        // finisher hand-off, 64 skip local band finishes, 128 skip split-band
                        // exchanges, 256 finisher folds without finishing, 8192 no
                        // launch-summary atomics,
                        // 1024 / 2048 force the contiguous / strided schedule
  const void* pred_in;  // [M] predicted row sums (fp32 (hi, lo) pairs) supplied by X's producer, or null
  int requant_shift;    // O_I8: the stored output's requantisation shift
  const void* residual; // ACT_RESIDUAL: [M, N] of the output type, stored = residual + y
  long long ld_res;
  int r_tma;            // 1: the residual is read through TMA boxes (tmR) into the staging boxes
  int replay;           // 1: only active bands, compare against old C
  int* changed;
  Workspace ws;
};

template <int KIND>
struct KindTraits;
template <>
struct KindTraits<K_BF16> {
  static constexpr int ELEM = 2;
  static constexpr int MMA_KIND = 0;
  static constexpr uint32_t IDESC = make_idesc(1, 1, BM, BN);
};
template <>
struct KindTraits<K_F16> {
  static constexpr int ELEM = 2;
  static constexpr int MMA_KIND = 0;
  static constexpr uint32_t IDESC = make_idesc(1, 0, BM, BN);
};
template <>
struct KindTraits<K_TF32> {
  static constexpr int ELEM = 4;
  static constexpr int MMA_KIND = 1;
  static constexpr uint32_t IDESC = make_idesc(1, 2, BM, BN);
};
template <>
struct KindTraits<K_I8> {
  static constexpr int ELEM = 1;
  static constexpr int MMA_KIND = 2;
  static constexpr uint32_t IDESC = make_idesc(2, 1, BM, BN);
};

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ float bf16_bits_to_f32(uint32_t b) { return __uint_as_float(b << 16); }
__device__ __forceinline__ float f16_bits_to_f32(uint32_t b) {
  return __half2float(__ushort_as_half(static_cast<unsigned short>(b)));
}

// Key for the "max over non-NaN |d - mu|" reduction: 0 = no non-NaN value;
// otherwise (bits of the non-negative double) + 1, which orders like the value.
__device__ __forceinline__ unsigned long long gap_key(double gap) {
  if (gap != gap) return 0ull;
  return static_cast<unsigned long long>(__double_as_longlong(gap)) + 1ull;
}

// ---- binary64 from integer arithmetic.  The kernels form d, its flag and its gap key
// without a single FP64 instruction: next to a busy tensor pipe each DADD / F2F.F64
// stalls the SM far beyond its count (a few dozen per band cost up to 18% of a
// 50432 x 4096 x 4096 launch).  d is computed in double-float (fp32 pairs, as the
// partial sums) and rounded once, to nearest-even, into binary64 bits.

// (hi, lo) + (hi, lo) fp32 pairs, hi in the low word; relative error ~2^-44.
__device__ __forceinline__ unsigned long long df_add(unsigned long long a, unsigned long long b) {
  const float ah = __uint_as_float(static_cast<uint32_t>(a)), al = __uint_as_float(static_cast<uint32_t>(a >> 32));
  const float bh = __uint_as_float(static_cast<uint32_t>(b)), bl = __uint_as_float(static_cast<uint32_t>(b >> 32));
  const float sh = ah + bh, bp = sh - ah;
  float e = (ah - (sh - bp)) + (bh - bp);
  e += al + bl;
  const float h = sh + e, l = e - (h - sh);
  return static_cast<unsigned long long>(__float_as_uint(h)) | (static_cast<unsigned long long>(__float_as_uint(l)) << 32);
}

// mag * 2^e2 (mag != 0, leading bit at p), rounded to nearest-even into binary64 bits;
// the callers keep the exponent inside the normal range.
__device__ __forceinline__ unsigned long long f64_bits_round(unsigned long long mag, int p, int e2, bool neg) {
  int ex = p + e2;
  unsigned long long keep;
  if (p > 52) {
    const int r = p - 52;
    keep = mag >> r;
    const unsigned long long rem = mag & ((1ull << r) - 1ull), half = 1ull << (r - 1);
    if (rem > half || (rem == half && (keep & 1ull))) ++keep;
    if (keep >> 53) {
      keep >>= 1;
      ++ex;
    }
  } else {
    keep = mag << (52 - p);
  }
  return (neg ? (1ull << 63) : 0ull) | (static_cast<unsigned long long>(ex + 1023) << 52) | (keep & ((1ull << 52) - 1ull));
}

__device__ __forceinline__ unsigned long long f64_bits_of_f32(uint32_t u) {
  const unsigned long long sg = static_cast<unsigned long long>(u >> 31) << 63;
  const uint32_t e = (u >> 23) & 0xffu, m = u & 0x7fffffu;
  if (e == 0xffu) return sg | 0x7ff0000000000000ull | (static_cast<unsigned long long>(m) << 29);
  if (e == 0u) return m == 0u ? sg : f64_bits_round(m, 31 - __clz(m), -149, sg != 0ull);
  return sg | (static_cast<unsigned long long>(e + 896u) << 52) | (static_cast<unsigned long long>(m) << 29);
}

__device__ __forceinline__ unsigned long long f64_bits_of_u64(unsigned long long v) {
  return v == 0ull ? 0ull : f64_bits_round(v, 63 - __clzll(static_cast<long long>(v)), 0, false);
}

// hi + lo of an fp32 pair, rounded once to binary64 (exact whenever it fits 53 bits).
// Out of line: the rare general case of f64_bits_of_df_norm (one copy, not one per row).
__device__ __noinline__ unsigned long long f64_bits_of_df(unsigned long long df) {
  const uint32_t uh = static_cast<uint32_t>(df), ul = static_cast<uint32_t>(df >> 32);
  const uint32_t eh = (uh >> 23) & 0xffu, el = (ul >> 23) & 0xffu;
  if (eh == 0xffu || el == 0xffu) return f64_bits_of_f32(__float_as_uint(__uint_as_float(uh) + __uint_as_float(ul)));
  if ((ul << 1) == 0u) return f64_bits_of_f32(uh);
  if ((uh << 1) == 0u) return f64_bits_of_f32(ul);
  unsigned long long ma = eh ? ((uh & 0x7fffffu) | 0x800000u) : (uh & 0x7fffffu);
  unsigned long long mb = el ? ((ul & 0x7fffffu) | 0x800000u) : (ul & 0x7fffffu);
  int ea = eh ? static_cast<int>(eh) - 150 : -149, eb = el ? static_cast<int>(el) - 150 : -149;
  bool na = (uh >> 31) != 0u, nb = (ul >> 31) != 0u;
  if (eb > ea) {
    const unsigned long long tm = ma; ma = mb; mb = tm;
    const int te = ea; ea = eb; eb = te;
    const bool tn = na; na = nb; nb = tn;
  }
  // fixed point with the larger operand's 24 bits at 61..38; the smaller one's bits
  // shifted out below bit 0 (only when it lies > 38 bits lower) are jammed into bit 0,
  // which sits at least 8 bits under the rounding position then
  const int sh = ea - eb;
  const unsigned long long X = ma << 38, Yf = mb << 38;
  const unsigned long long Y = sh >= 64 ? 0ull : (Yf >> sh);
  const bool sticky = sh >= 64 ? true : (Yf & ((1ull << sh) - 1ull)) != 0ull;
  unsigned long long mag;
  bool neg;
  if (na == nb) {
    mag = (X + Y) | (sticky ? 1ull : 0ull);
    neg = na;
  } else if (!sticky) {
    neg = X >= Y ? na : nb;
    mag = X >= Y ? X - Y : Y - X;
  } else {  // X > Y here
    mag = (X - Y - 1ull) | 1ull;
    neg = na;
  }
  if (mag == 0ull) return 0ull;
  return f64_bits_round(mag, 63 - __clzll(static_cast<long long>(mag)), ea - 38, neg);
}

// The same for a pair from df_add (|lo| <= ulp32(hi) / 2): double(hi) stepped by lo in
// units of hi's binary64 ulp (half that when hi is a power of two and lo points down,
// the one case that leaves hi's binade); one F2I with round-to-nearest-even is the
// tie rule, since double(hi)'s low 29 bits are zero.  |hi| < 2^-75, non-finite or
// unnormalised pairs take the general routine.
__device__ __forceinline__ unsigned long long f64_bits_of_df_norm(unsigned long long df) {
  const uint32_t uh = static_cast<uint32_t>(df), ul = static_cast<uint32_t>(df >> 32);
  const uint32_t eh = (uh >> 23) & 0xffu;
  if (eh >= 52u && eh <= 254u) {
    const uint32_t mh = uh & 0x7fffffu;
    const bool down = ((uh ^ ul) >> 31) != 0u && (ul << 1) != 0u;  // lo shrinks |hi|
    const uint32_t s = 306u - eh + ((mh == 0u && down) ? 1u : 0u);  // float 2^(s-127) = 1 / ulp
    const float scaled = __uint_as_float(ul) * __uint_as_float(s << 23);
    const int L = __float2int_rn(scaled);
    if (L >= -(1 << 29) && L <= (1 << 29)) {
      const unsigned long long D =
          (static_cast<unsigned long long>(uh >> 31) << 63) | (static_cast<unsigned long long>(eh + 896u) << 52) |
          (static_cast<unsigned long long>(mh) << 29);
      return (uh >> 31) ? D - static_cast<unsigned long long>(static_cast<long long>(L))
                        : D + static_cast<unsigned long long>(static_cast<long long>(L));
    }
  }
  return f64_bits_of_df(df);
}

// Order-preserving key of binary64 bits (+0 and -0 equal); NaNs are screened by the caller.
__host__ __device__ __forceinline__ unsigned long long f64_order_key(unsigned long long b) {
  if ((b << 1) == 0ull) b = 0ull;
  return (b >> 63) ? ~b : (b | (1ull << 63));
}
__host__ __device__ __forceinline__ bool f64_bits_nan(unsigned long long b) {
  return (b & 0x7fffffffffffffffull) > 0x7ff0000000000000ull;
}

template <int OUT>
__device__ __forceinline__ uint32_t load_out_bits(const void* base, long long idx) {
  if constexpr (OUT == O_BF16 || OUT == O_F16)
    return static_cast<const unsigned short*>(base)[idx];
  else
    return static_cast<const uint32_t*>(base)[idx];
}
template <int OUT>
__device__ __forceinline__ void store_out_bits(void* base, long long idx, uint32_t bits) {
  if constexpr (OUT == O_BF16 || OUT == O_F16)
    static_cast<unsigned short*>(base)[idx] = static_cast<unsigned short>(bits);
  else
    static_cast<uint32_t*>(base)[idx] = bits;
}
template <int OUT>
__device__ __forceinline__ double out_bits_to_f64(uint32_t b) {
  if constexpr (OUT == O_BF16) return static_cast<double>(bf16_bits_to_f32(b));
  else if constexpr (OUT == O_F16) return static_cast<double>(f16_bits_to_f32(b));
  else if constexpr (OUT == O_F32) return static_cast<double>(__uint_as_float(b));
  else return static_cast<double>(static_cast<int>(b));
}
// accumulator (+bias) -> stored encoding, round to nearest even
template <int OUT>
__device__ __forceinline__ uint32_t acc_to_out_bits(uint32_t acc, uint32_t bias_bits) {
  if constexpr (OUT == O_I32 || OUT == O_I8) {
    return acc + bias_bits;  // int32 wrap-around, numerics.py:269-272
  } else {
    const float v = __uint_as_float(acc) + __uint_as_float(bias_bits);
    if constexpr (OUT == O_BF16) return static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(v)));
    else if constexpr (OUT == O_F16) return static_cast<uint32_t>(__half_as_ushort(__float2half_rn(v)));
    else return __float_as_uint(v);
  }
}
template <int OUT>
__device__ __forceinline__ uint32_t value_to_out_bits(double v) {
  if constexpr (OUT == O_BF16) return static_cast<uint32_t>(__bfloat16_as_ushort(__double2bfloat16(v)));
  else if constexpr (OUT == O_F16) return static_cast<uint32_t>(__half_as_ushort(__double2half(v)));
  else if constexpr (OUT == O_F32) return __float_as_uint(__double2float_rn(v));
  else return static_cast<uint32_t>(static_cast<int>(static_cast<long long>(v)));
}
template <int OUT>
__device__ __forceinline__ uint32_t out_bits_mask() {
  if constexpr (OUT == O_BF16 || OUT == O_F16) return 0xFFFFu;
  else return 0xFFFFFFFFu;
}

// ======================================================================
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr)
               : "memory");
  return v;
}

}  // namespace gg
