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
enum : int { O_BF16 = 0, O_F16 = 1, O_F32 = 2, O_I32 = 3 };

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
  int one_tile;         // <= 1 tile per pair: split bands fold from one burst into the idle stages
  int dbg;              // diagnostics only ($GG_DEBUG), 0 in production: 1 skip predicted dot products,
                        // 2 decouple the checksum warps from the stages, 4 skip band folds, 8 skip
                        // observed sums, 64 skip local band finishes, 128 skip split-band exchanges,
                        // 1024 / 2048 force the contiguous / strided schedule
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
  if constexpr (OUT == O_I32) {
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
