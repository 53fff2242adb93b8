// gg_gemm_sm100.cuh — K1/K4: checksum-protected GEMM for sm_100a.
//
//   C[m, n] = sum_k A[m, k] * B[n, k] + bias[n]          (tcgen05, TMEM acc)
//   d[m]    = (sum_k A[m, k] * w_sum[k] + bias_sum) - sum_n C[m, n]
//   flags   = guard._verify_arrays rule on d            (guard.py:188-215)
//
// One persistent CTA per SM, warp-specialised (384 threads):
//   warp 0      TMA producer (A and B K-major tiles, 128B swizzle, 4 stages)
//   warp 1      tcgen05.mma issuer (one thread), accumulators in TMEM,
//               two 128x256 fp32/s32 buffers (512 columns) so the epilogue of
//               tile i overlaps the mainloop of tile i+1
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: tcgen05.ld one accumulator row per thread, bias,
//               round to the output type, fault injection, store, and the
//               OBSERVED row sum over the stored values (guard.py:170)
//   warps 8-11  checksum producer side: read the A stages from shared memory
//               as they stream past the MMA and form PREDICTED[m] =
//               A[m,:] . w_sum (guard.py:168-169) in fp64 (int64 for int8) —
//               no extra pass over X in HBM; K-blocks are dealt round-robin
//               over the band's N-tiles.
// Per M-band, the last of the 2*n_tiles contributions folds the per-tile
// observed and predicted partials in ascending tile order, forms d, flags and per-band
// summaries; the last band forms the launch summaries (nflag, triggered,
// max_disc) and resets the counters.  Everything is deterministic: no atomics
// touch C or d, so a recompute is byte-identical (needed by replay,
// guard.py:590).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "gg_sm100.cuh"
#include "../../include/gemmguard_b200.h"

namespace gg {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK_BYTES = 128;  // one 128B swizzle atom of K per stage
constexpr int STAGES = 4;
constexpr int THREADS = 384;
constexpr int A_STAGE_BYTES = BM * BK_BYTES;  // 16 KB
constexpr int B_STAGE_BYTES = BN * BK_BYTES;  // 32 KB
constexpr int TMEM_COLS = 2 * BN;             // two accumulator buffers
constexpr int SMEM_BYTES = STAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + 1024 /*align*/ + 256 /*barriers*/;

// operand kinds (template KIND)
enum : int { K_BF16 = 0, K_F16 = 1, K_TF32 = 2, K_I8 = 3 };
// output kinds (template OUT)
enum : int { O_BF16 = 0, O_F16 = 1, O_F32 = 2, O_I32 = 3 };

struct Workspace {
  int* counters;        // [0] done bands, [1] active bands
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
  void* C;
  long long ldc;
  const void* bias;
  // checksum
  const void* w_sum;    // f64 or i64
  const void* w_aux;    // bf16/f16: float2 (hi, lo) split of w_sum; i8: int32x4 signed digit planes
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

// 128-thread group reductions (named barrier `bar`, scratch in smem).
__device__ __forceinline__ int group_sum_i32(int v, int tid, uint32_t bar, int* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((tid & 31) == 0) scratch[tid >> 5] = v;
  named_bar_sync(bar, 128);
  int r = scratch[0] + scratch[1] + scratch[2] + scratch[3];
  named_bar_sync(bar, 128);
  return r;
}
__device__ __forceinline__ unsigned long long group_max_u64(unsigned long long v, int tid, uint32_t bar,
                                                            unsigned long long* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  if ((tid & 31) == 0) scratch[tid >> 5] = v;
  named_bar_sync(bar, 128);
  unsigned long long r = scratch[0];
#pragma unroll
  for (int i = 1; i < 4; ++i) r = scratch[i] > r ? scratch[i] : r;
  named_bar_sync(bar, 128);
  return r;
}
__device__ __forceinline__ double group_sum_f64_fixed(double v, int tid, uint32_t bar, double* scratch) {
  // fixed-order tree: deterministic for a fixed thread->value assignment
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((tid & 31) == 0) scratch[tid >> 5] = v;
  named_bar_sync(bar, 128);
  double r = (scratch[0] + scratch[1]) + (scratch[2] + scratch[3]);
  named_bar_sync(bar, 128);
  return r;
}

struct GroupScratch {
  int flag;
  int isum[4];
  unsigned long long umax[4];
  double dsum[4];
};

// Called by a 128-thread group (epilogue or checksum side) after it has
// published its contribution to band m.  The last contributor finalises the
// band; the last band finalises the launch.
template <bool INT>
__device__ void band_arrive(const Params& p, int m, int tid, uint32_t bar, GroupScratch* gs) {
  // Release: every thread fences its own partial write (a fence orders only
  // the calling thread's writes), then thread 0 counts the contribution.
  __threadfence();
  named_bar_sync(bar, 128);
  if (tid == 0) {
    const int old = atomicAdd(&p.ws.band_counter[m], 1);
    gs->flag = (old == 2 * p.n_tiles - 1) ? 1 : 0;  // n_tiles observed + n_tiles predicted partials
    if (gs->flag) __threadfence();                  // acquire the other contributions
  }
  named_bar_sync(bar, 128);
  if (!gs->flag) return;

  // ---- finalise band m: d, flags, band summaries (fixed ascending tile order)
  const int row = m * BM + tid;
  int nflag = 0;
  unsigned long long key = 0;
  if (row < p.M) {
    bool flag;
    if constexpr (INT) {
      long long obs = 0, pred = 0;
      const long long* part = reinterpret_cast<const long long*>(p.ws.partial);
      const long long* predp = reinterpret_cast<const long long*>(p.ws.pred);
      for (int t = 0; t < p.n_tiles; ++t) {
        obs += __ldcg(&part[(size_t)t * p.m_pad + row]);
        pred += __ldcg(&predp[(size_t)t * p.m_pad + row]);
      }
      const long long di = (pred + p.bias_sum_i) - obs;
      static_cast<long long*>(p.d)[row] = di;
      flag = di != 0;
      const unsigned long long mag = di < 0 ? 0ull - static_cast<unsigned long long>(di) : static_cast<unsigned long long>(di);
      key = gap_key(static_cast<double>(mag));
    } else {
      double obs = 0.0, pred = 0.0;
      for (int t = 0; t < p.n_tiles; ++t) {
        obs += ldcg_f64(&p.ws.partial[(size_t)t * p.m_pad + row]);
        pred += ldcg_f64(&p.ws.pred[(size_t)t * p.m_pad + row]);
      }
      const double dd = (pred + p.bias_sum_f) - obs;
      static_cast<double*>(p.d)[row] = dd;
      flag = !((dd >= p.lo) && (dd <= p.hi));
      key = gap_key(fabs(dd - p.mu));
    }
    if (INT || p.statistic == GG_PER_SAMPLE) {
      p.flags[row] = flag ? 1 : 0;
      nflag = flag ? 1 : 0;
    }
  }
  nflag = group_sum_i32(nflag, tid, bar, gs->isum);
  key = group_max_u64(key, tid, bar, gs->umax);
  __threadfence();  // d / flags of this band, before the launch-level count
  named_bar_sync(bar, 128);
  if (tid == 0) {
    p.ws.band_nflag[m] = nflag;
    p.ws.band_maxkey[m] = key;
    p.ws.band_counter[m] = 0;
    __threadfence();
    const int total = p.replay ? __ldcg(&p.ws.counters[1]) : p.m_tiles;
    const int old = atomicAdd(&p.ws.counters[0], 1);
    gs->flag = (old == total - 1) ? 1 : 0;
    if (gs->flag) __threadfence();
  }
  named_bar_sync(bar, 128);
  if (!gs->flag) return;

  // ---- last band: launch summaries over ALL bands (replayed or not)
  int nf = 0;
  unsigned long long mk = 0;
  for (int b = tid; b < p.m_tiles; b += 128) {
    nf += __ldcg(&p.ws.band_nflag[b]);
    unsigned long long k = __ldcg(&p.ws.band_maxkey[b]);
    mk = k > mk ? k : mk;
  }
  nf = group_sum_i32(nf, tid, bar, gs->isum);
  mk = group_max_u64(mk, tid, bar, gs->umax);
  if (!INT && p.statistic == GG_BATCH_MEAN) {
    // mean(d) over all rows in a fixed order; every row flags iff outside
    double s = 0.0;
    for (int r = tid; r < p.M; r += 128) s += ldcg_f64(&static_cast<double*>(p.d)[r]);
    s = group_sum_f64_fixed(s, tid, bar, gs->dsum);
    const double dm = s / static_cast<double>(p.M);
    const bool inside = (p.lo <= dm) && (dm <= p.hi);
    for (int r = tid; r < p.M; r += 128) p.flags[r] = inside ? 0 : 1;
    nf = inside ? 0 : p.M;
  }
  if (tid == 0) {
    *p.nflag = nf;
    *p.triggered = nf > 0 ? 1 : 0;
    *p.max_disc = (mk == 0ull) ? __longlong_as_double(0x7FF0000000000000ll)
                               : __longlong_as_double(static_cast<long long>(mk - 1ull));
    p.ws.counters[0] = 0;
    __threadfence();
  }
}

// Store 32 outputs of one row chunk (fast path: full chunk, aligned).
template <int OUT>
__device__ __forceinline__ void store_chunk_vec(void* cptr, const uint32_t (&o)[32]) {
  if constexpr (OUT == O_BF16 || OUT == O_F16) {
    uint4* dst = reinterpret_cast<uint4*>(cptr);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 v;
      v.x = (o[8 * q + 0] & 0xFFFFu) | (o[8 * q + 1] << 16);
      v.y = (o[8 * q + 2] & 0xFFFFu) | (o[8 * q + 3] << 16);
      v.z = (o[8 * q + 4] & 0xFFFFu) | (o[8 * q + 5] << 16);
      v.w = (o[8 * q + 6] & 0xFFFFu) | (o[8 * q + 7] << 16);
      dst[q] = v;
    }
  } else {
    uint4* dst = reinterpret_cast<uint4*>(cptr);
#pragma unroll
    for (int q = 0; q < 8; ++q) dst[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
  }
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

// Tile t -> (m, n), N-tile fastest: the n_tiles tiles of one M-band run on
// neighbouring CTAs at the same time, so each A band is read from HBM once
// and B (the weight) stays L2-resident.
__device__ __forceinline__ void tile_coords(const Params& p, int t, int& m, int& n) {
  m = t / p.n_tiles;
  n = t - m * p.n_tiles;
}

template <int KIND, int OUT, bool PROTECT>
__global__ void __launch_bounds__(THREADS, 1)
    gg_protected_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                             const Params p) {
  using T = KindTraits<KIND>;
  constexpr bool INT = (KIND == K_I8);
  constexpr int BK = BK_BYTES / T::ELEM;            // elements of K per stage
  constexpr int MMA_K_BYTES = 32;                   // K bytes per tcgen05.mma
  constexpr int MMAS_PER_STAGE = BK_BYTES / MMA_K_BYTES;
  constexpr int OUT_BYTES = (OUT == O_BF16 || OUT == O_F16) ? 2 : 4;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES * A_STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smB + STAGES * B_STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  __shared__ GroupScratch gscratch[2];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_tiles = p.m_tiles * p.n_tiles;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], PROTECT ? 1 + 4 : 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 4);
    }
    fence_barrier_init();
    fence_proxy_async_smem();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto tile_active = [&](int m) -> bool { return !p.replay || p.ws.band_active[m] != 0; };

  if (warp == 0) {
    // ================================================= TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int m, n;
        tile_coords(p, t, m, n);
        if (!tile_active(m)) continue;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], A_STAGE_BYTES + B_STAGE_BYTES);
          tma_load_2d(smA + stage * A_STAGE_BYTES, &tmA, &full_bar[stage], kb * BK, m * BM);
          tma_load_2d(smB + stage * B_STAGE_BYTES, &tmB, &full_bar[stage], kb * BK, n * BN);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ================================================= MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int m, n;
        tile_coords(p, t, m, n);
        if (!tile_active(m)) continue;
        const int buf = local & 1;
        const uint32_t use = static_cast<uint32_t>(local >> 1);
        mbar_wait(&tempty_bar[buf], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(buf * BN);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t adesc = sw128_kmajor_desc(smem_u32(smA + stage * A_STAGE_BYTES));
          const uint64_t bdesc = sw128_kmajor_desc(smem_u32(smB + stage * B_STAGE_BYTES));
#pragma unroll
          for (int kk = 0; kk < MMAS_PER_STAGE; ++kk) {
            // advance the start address by 32 B (>>4 = 2) per K step inside the atom
            tc_mma<T::MMA_KIND>(d_tmem, adesc + static_cast<uint64_t>(kk * (MMA_K_BYTES >> 4)),
                                bdesc + static_cast<uint64_t>(kk * (MMA_K_BYTES >> 4)), T::IDESC,
                                (kb | kk) != 0 ? 1u : 0u);
          }
          tc_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull_bar[buf]);
        ++local;
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ================================================= epilogue
    const int eg = warp - 4;           // TMEM lane group == warp % 4
    const int tid = threadIdx.x - 128; // 0..127 == accumulator row in tile
    const bool vec_ok = ((p.ldc * OUT_BYTES) % 16 == 0) && ((reinterpret_cast<uintptr_t>(p.C) & 15) == 0);
    const bool bias_vec = (p.bias != nullptr) && ((p.N & 3) == 0) && ((reinterpret_cast<uintptr_t>(p.bias) & 15) == 0);
    int local = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int m, n;
      tile_coords(p, t, m, n);
      if (!tile_active(m)) continue;
      const int buf = local & 1;
      const uint32_t use = static_cast<uint32_t>(local >> 1);
      mbar_wait(&tfull_bar[buf], use & 1);
      tc_fence_after();
      const int row = m * BM + tid;
      const bool row_ok = row < p.M;
      const int n0 = n * BN;
      const int nchunks = min(BN / 32, (p.N - n0 + 31) / 32);  // chunks holding valid columns
      double obs = 0.0;      // float kinds
      long long obs_i = 0;   // int kind (exact)
      int changed = 0;
#pragma unroll 1
      for (int c = 0; c < nchunks; ++c) {
        const int col0 = n0 + 32 * c;
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(eg * 32) << 16) + static_cast<uint32_t>(buf * BN + 32 * c), r);
        tmem_ld_wait();
        if (c == nchunks - 1) {
          // all TMEM reads of this buffer are done: hand it back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[buf]);
        }
        const bool full = (col0 + 32 <= p.N);
        // faults on this row inside this chunk (rare; the list is short)
        for (int i = 0; i < p.n_inj; ++i) {
          const gg_injection f = p.inj[i];
          if (f.row == row && f.target == GG_INJ_ACCUMULATOR && f.col >= col0 && f.col < col0 + 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (f.col == col0 + j) r[j] ^= (1u << (f.bit & 31));
          }
        }
        uint32_t o[32];
        if (full && bias_vec) {
          const uint4* bp = reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(p.bias) + col0);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint4 bv = __ldg(bp + q);
            o[4 * q + 0] = acc_to_out_bits<OUT>(r[4 * q + 0], bv.x);
            o[4 * q + 1] = acc_to_out_bits<OUT>(r[4 * q + 1], bv.y);
            o[4 * q + 2] = acc_to_out_bits<OUT>(r[4 * q + 2], bv.z);
            o[4 * q + 3] = acc_to_out_bits<OUT>(r[4 * q + 3], bv.w);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const uint32_t bj =
                (p.bias != nullptr && col0 + j < p.N) ? __ldg(static_cast<const uint32_t*>(p.bias) + col0 + j) : 0u;
            o[j] = acc_to_out_bits<OUT>(r[j], bj);
          }
        }
        for (int i = 0; i < p.n_inj; ++i) {
          const gg_injection f = p.inj[i];
          if (f.row == row && f.target == GG_INJ_OUTPUT && f.col >= col0 && f.col < col0 + 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (f.col == col0 + j)
                o[j] = (f.mode == GG_INJ_BITFLIP) ? ((o[j] ^ (1u << (f.bit & 31))) & out_bits_mask<OUT>())
                                                  : value_to_out_bits<OUT>(f.value);
          }
        }
        if (row_ok) {
          const long long base = static_cast<long long>(row) * p.ldc + col0;
          if (p.replay) {
            for (int j = 0; j < 32; ++j)
              if (col0 + j < p.N) changed += (load_out_bits<OUT>(p.C, base + j) != o[j]) ? 1 : 0;
          }
          if (full && vec_ok) {
            store_chunk_vec<OUT>(static_cast<uint8_t*>(p.C) + base * OUT_BYTES, o);
          } else {
            for (int j = 0; j < 32; ++j)
              if (col0 + j < p.N) store_out_bits<OUT>(p.C, base + j, o[j]);
          }
          if constexpr (PROTECT) {
            // observed row sum of the STORED values (guard.py:170)
            if constexpr (INT) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (full || col0 + j < p.N) obs_i += static_cast<long long>(static_cast<int>(o[j]));
            } else if constexpr (OUT == O_F32) {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (full || col0 + j < p.N) obs += static_cast<double>(__uint_as_float(o[j]));
            } else {
              // 16-bit outputs are exact in fp32; fold groups of 8 in fp32, then fp64
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                float s8 = 0.f;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  const int j = 8 * g + e;
                  const float yv = (OUT == O_BF16) ? bf16_bits_to_f32(o[j]) : f16_bits_to_f32(o[j]);
                  s8 += (full || col0 + j < p.N) ? yv : 0.f;
                }
                obs += static_cast<double>(s8);
              }
            }
          }
        }
      }
      if (nchunks <= 0) {  // cannot happen for n < n_tiles; keep the handshake total
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[buf]);
      }
      if (p.replay && p.changed != nullptr) {
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) changed += __shfl_xor_sync(0xffffffffu, changed, o2);
        if (lane == 0 && changed) atomicAdd(p.changed, changed);
      }
      if constexpr (PROTECT) {
        if (row_ok) {
          if constexpr (INT) reinterpret_cast<long long*>(p.ws.partial)[static_cast<size_t>(n) * p.m_pad + row] = obs_i;
          else p.ws.partial[static_cast<size_t>(n) * p.m_pad + row] = obs;
        }
        band_arrive<INT>(p, m, tid, 1, &gscratch[0]);
      }
      ++local;
    }
  } else if (warp >= 8) {
    // ================================================= checksum producer side
    // PREDICTED[m] = sum_k A[m,k] * w_sum[k] (guard.py:168-169), read from the
    // A stages in shared memory.  The K-blocks of a band are dealt round-robin
    // to the band's N-tiles (tile n takes kb % n_tiles == n), so every tile
    // carries 1/n_tiles of the side work and no stage is held long.
    if constexpr (PROTECT) {
      const int tid = threadIdx.x - 256;  // 0..127 == row in tile
      const int sw = tid & 7;
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int m, n;
        tile_coords(p, t, m, n);
        if (!tile_active(m)) continue;
        double accd = 0.0;                 // bf16/f16/tf32
        int acc8[3] = {0, 0, 0};           // int8 digit planes (exact)
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          const bool mine = (kb % p.n_tiles) == n;
          uint4 v[8];
          if (mine) {
            // copy this row's 128 B of the stage to registers, then release
            const uint32_t rowaddr = smem_u32(smA + stage * A_STAGE_BYTES) + static_cast<uint32_t>(tid * 128);
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = lds128(rowaddr + static_cast<uint32_t>((j ^ sw) << 4));
            // WAR across proxies: these generic-proxy reads must be ordered before
            // the async-proxy (TMA) refill the empty-barrier arrival enables.
            fence_proxy_async_smem();
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          if (!mine) continue;
          const int kbase = kb * BK;
          const bool tail = kbase + BK > p.K;  // warp-uniform; TMA zero-fills x beyond K
          if constexpr (INT) {
            // sum_k x*w = sum_d 256^d * sum_k x*digit_d(w): IDP4A, exact in int32
            const int4* dig = static_cast<const int4*>(p.w_aux) + (kbase >> 2);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint32_t w4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int kq = kbase + j * 16 + q * 4;
                int4 dd = make_int4(0, 0, 0, 0);
                if (!tail || kq < p.K) dd = __ldg(dig + j * 4 + q);
                acc8[0] = __dp4a(static_cast<int>(w4[q]), dd.x, acc8[0]);
                acc8[1] = __dp4a(static_cast<int>(w4[q]), dd.y, acc8[1]);
                acc8[2] = __dp4a(static_cast<int>(w4[q]), dd.z, acc8[2]);
              }
            }
          } else if constexpr (KIND == K_TF32) {
            // fp32 operands: full fp64 products (x exact in double)
            const double* wf = static_cast<const double*>(p.w_sum);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const uint32_t w4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int k = kbase + j * 4 + e;
                const double w = (!tail || k < p.K) ? __ldg(wf + k) : 0.0;
                accd = fma(static_cast<double>(__uint_as_float(w4[e])), w, accd);
              }
            }
          } else {
            // bf16/f16: x is exact in fp32; w_sum = hi + lo (two fp32); fp32 FMAs
            // over 16-element groups, folded into fp64 once per group.
            const float2* w2 = static_cast<const float2*>(p.w_aux) + kbase;
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              float sh = 0.f, sl = 0.f;
#pragma unroll
              for (int jj = 0; jj < 2; ++jj) {
                const int j = 2 * g + jj;
                const uint32_t w4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  const int k = j * 8 + e;
                  const uint32_t h = (w4[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
                  float x;
                  if constexpr (KIND == K_BF16) x = bf16_bits_to_f32(h);
                  else x = f16_bits_to_f32(h);
                  float2 w = make_float2(0.f, 0.f);
                  if (!tail || kbase + k < p.K) w = __ldg(w2 + k);
                  sh = fmaf(x, w.x, sh);
                  sl = fmaf(x, w.y, sl);
                }
              }
              accd += static_cast<double>(sh);
              accd += static_cast<double>(sl);
            }
          }
        }
        const int row = m * BM + tid;
        if (row < p.M) {
          if constexpr (INT) {
            const long long pr = static_cast<long long>(acc8[0]) + 256ll * acc8[1] + 65536ll * acc8[2];
            reinterpret_cast<long long*>(p.ws.pred)[static_cast<size_t>(n) * p.m_pad + row] = pr;
          } else {
            p.ws.pred[static_cast<size_t>(n) * p.m_pad + row] = accd;
          }
        }
        band_arrive<INT>(p, m, tid, 2, &gscratch[1]);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, TMEM_COLS);
}

}  // namespace gg
