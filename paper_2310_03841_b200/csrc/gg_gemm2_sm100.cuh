// gg_gemm2_sm100.cuh — K1/K4: checksum-protected GEMM on CTA pairs (sm_100a).
//
//   C[m, n] = sum_k A[m, k] * B[n, k] + bias[n]          (tcgen05.mma.cta_group::2)
//   d[m]    = (sum_k A[m, k] * w_sum[k] + bias_sum) - sum_n C[m, n]
//   flags   = guard._verify_arrays rule on d            (guard.py:188-215)
//
// A cluster of two CTAs on the two SMs of a TPC computes 256 x 256 tiles: each
// CTA stages 128 rows of A and 128 rows (N) of B per K-block, the leader issues
// one M=256, N=256 MMA reading both CTAs' shared memory, and each CTA's TMEM
// holds the fp32/s32 accumulators of its own 128 rows (two 256-column buffers:
// the epilogue of tile i overlaps the mainloop of tile i+1).
//
// Tile schedule: the pair tiles (256-row band m, 256-column tile n; n fastest)
// are cut into one CONTIGUOUS range per pair, so a pair walks whole row bands
// and folds their checksums locally; only a band cut by a range boundary
// exchanges partials through global memory.  When the A bands streamed by all
// pairs at once would not fit in L2 (long K), pairs walk the tiles strided
// instead (neighbouring pairs share A bands in L2) and every band exchanges
// its partials through global memory.
//
// Warp roles (512 threads per CTA).  The SMSP arbiter issues the highest
// warp id first, so ids follow criticality:
//   15     MMA issuer (leader only, one thread): stage release and accumulator
//          hand-off are tcgen05.commit multicasts to both CTAs; relays "owned
//          stage landed" to both CTAs' checksum warps before issuing its MMAs
//   14     TMA producer (both CTAs; loads complete on the LEADER's full barrier)
//   13     TMEM allocator (both CTAs, cta_group::2)
//   12     reducer: folds the per-tile row partials of each band (registers
//          for local bands, global partials + one fence for split bands),
//          writes d / flags and the launch summaries
//   8-11   checksum producer side: PREDICTED[m] = A[m,:] . w_sum (guard.py:
//          168-169) from the A stages already in shared memory, w from shared
//          memory.  A band's K-blocks are dealt round-robin over its N-tiles;
//          the checksum warps copy their row of an owned stage to registers
//          and release it at once.
//   0-7    epilogue, two warps per TMEM lane quadrant (warp % 4), each owning
//          half of the tile's columns: TMEM -> registers, bias, round, fault
//          injection, OBSERVED row sums over the stored values (guard.py:170),
//          then a 32x32 swizzled smem box per warp and a TMA store.
// Everything is deterministic (fixed fold orders, no float atomics), so a
// recompute is byte-identical — required by replay (guard.py:590).
#pragma once
#include "gg_gemm_sm100.cuh"

namespace gg {
namespace pair {

// Diagnostics: with -DGG_TRACE the roles stamp clock64() per tile into a
// device buffer (gg_trace_buffer); compiled out of the production library.
#ifdef GG_TRACE
__device__ unsigned long long* g_trace = nullptr;
constexpr int TRACE_TILES = 64, TRACE_EV = 28;
#define GG_EV(ev, local)                                                                                  \
  do {                                                                                                  \
    if (g_trace != nullptr && (local) < TRACE_TILES)                                                    \
      g_trace[(static_cast<size_t>(blockIdx.x) * TRACE_TILES + (local)) * TRACE_EV + (ev)] = clock64(); \
  } while (0)
#else
#define GG_EV(ev, local) \
  do {                   \
  } while (0)
#endif

// Diagnostic switches ($GG_DEBUG, Params::dbg) exist only in diagnostics builds
// (python -m paper_2310_03841_b200.build --trace / --variant diag GG_DIAGNOSTICS).
#ifdef GG_DIAGNOSTICS
#define GG_DBG(bit) ((p.dbg & (bit)) != 0)
#else
#define GG_DBG(bit) false
#endif

constexpr int BM = 128;           // rows per CTA (256 per pair)
constexpr int BN = 256;           // MMA N per tile; each CTA stages BN/2 rows of B
constexpr int BK_BYTES = 128;     // one 128 B swizzle atom of K per stage
constexpr int STAGES = 5;
constexpr int THREADS = 512;
constexpr int A_BYTES = BM * BK_BYTES;        // 16 KB
constexpr int B_BYTES = (BN / 2) * BK_BYTES;  // 16 KB
constexpr int TMEM_COLS = 2 * BN;
constexpr int EPI_WARPS = 8;                 // two per TMEM lane quadrant, each owning half the columns
constexpr int CBOX = 32;                      // epilogue store box: 32 rows x 32 columns
constexpr int CST_BYTES = 4096;               // staging per epilogue warp: 2 x 2 KB boxes (16-bit out) or 1 x 4 KB
constexpr int C_OFF = STAGES * (A_BYTES + B_BYTES);
constexpr int BAR_OFF = C_OFF + EPI_WARPS * CST_BYTES;
constexpr int NSLOT = 4;                      // depth of the observed / predicted partial rings
// finisher queue: split bands whose fold the reducer hands off.  Deep enough that the
// reducer never waits on it: a reducer held up here arrives last at its next bands'
// counters too, which hands it their folds as well (a feedback loop that left single
// CTAs tens of microseconds behind on long-N shapes).
constexpr int FQ = 16;
constexpr int QAREA = (16 + 4 * FQ + 15) / 16 * 16;  // tmem slot + queued band ids
constexpr int NBAR = 4 * STAGES + 4 + 4 * NSLOT + 2 * FQ + 2 * EPI_WARPS;  // + the residual boxes' loads
constexpr int W_SMEM = 16384;                 // checksum w-vector kept in shared memory when it fits
constexpr int SMEM_BYTES = BAR_OFF + NBAR * 8 + QAREA /*tmem slot, finisher queue*/ + 3 * NSLOT * BM * 8 /*partial rings*/ +
                           2 * BN * 4 /*bias tiles*/ + W_SMEM + 1024 /*align*/;

template <int KIND> struct PairIdesc;
template <> struct PairIdesc<K_BF16> { static constexpr uint32_t V = make_idesc(1, 1, 256, BN); };
template <> struct PairIdesc<K_F16> { static constexpr uint32_t V = make_idesc(1, 0, 256, BN); };
template <> struct PairIdesc<K_TF32> { static constexpr uint32_t V = make_idesc(1, 2, 256, BN); };
template <> struct PairIdesc<K_I8> { static constexpr uint32_t V = make_idesc(2, 1, 256, BN); };

// Contiguous tile range of pair `pid` out of `npairs` over `total` tiles.
__device__ __forceinline__ void pair_range(int pid, int npairs, int total, int& t0, int& t1) {
  t0 = static_cast<int>(static_cast<long long>(pid) * total / npairs);
  t1 = static_cast<int>(static_cast<long long>(pid + 1) * total / npairs);
}

// d / flag / gap key of one row from its folded sums (guard.py:163-171, 188-215).  Flags follow
// the per-sample rule; a batch_mean launch has its flags re-derived from every d by the
// launcher's follow-up pass (NumPy's pairwise mean, guard.py:198-201).
template <bool INT>
__device__ __forceinline__ void row_check(const Params& p, unsigned long long obs, unsigned long long pred,
                                          unsigned long long& dbits, bool& flag, unsigned long long& key) {
  if constexpr (INT) {
    const long long di = (static_cast<long long>(pred) + p.bias_sum_i) - static_cast<long long>(obs);
    dbits = static_cast<unsigned long long>(di);
    flag = di != 0;
    const unsigned long long mag =
        di < 0 ? 0ull - static_cast<unsigned long long>(di) : static_cast<unsigned long long>(di);
    key = f64_bits_of_u64(mag) + 1ull;  // gap_key(double(|d|))
  } else {
    // d = (pred + bias) - obs in double-float, one rounding to binary64 (no FP64 instruction)
    const unsigned long long dd = df_add(df_add(pred, p.bias_df), obs ^ 0x8000000080000000ull);
    const unsigned long long db = f64_bits_of_df_norm(dd);
    dbits = db;
    const unsigned long long ok = f64_order_key(db);
    flag = f64_bits_nan(db) || ok < p.lo_key || ok > p.hi_key;  // !(lo <= d <= hi)
    unsigned long long gb = db & 0x7fffffffffffffffull;         // |d - mu|
    if (!p.mu_zero) {
      unsigned long long g = df_add(dd, p.neg_mu_df);
      if (static_cast<uint32_t>(g) >> 31) g ^= 0x8000000080000000ull;
      gb = f64_bits_of_df_norm(g);
    }
    key = f64_bits_nan(gb) ? 0ull : gb + 1ull;  // gap_key
  }
}

// d / flags of the rows lane + 32q (q < 4) of band mb from their folded sums, with the
// band's flag count and largest gap key reduced over the warp (no stores).
template <bool INT>
struct BandRows {
  unsigned long long dbits[4];  // d (f64 or i64 bits)
  bool flag[4];
  int nflag;
  unsigned long long key;
};

template <bool INT>
__device__ __forceinline__ BandRows<INT> band_rows(const Params& p, int mb, int lane, const unsigned long long (&obs)[4],
                                                  const unsigned long long (&pred)[4]) {
  BandRows<INT> r;
  r.nflag = 0;
  r.key = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int row = mb * BM + lane + 32 * q;
    r.flag[q] = false;
    r.dbits[q] = 0;
    if (row >= p.M) continue;
    unsigned long long k;
    row_check<INT>(p, obs[q], pred[q], r.dbits[q], r.flag[q], k);
    r.key = k > r.key ? k : r.key;
    r.nflag += r.flag[q] ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r.nflag += __shfl_xor_sync(0xffffffffu, r.nflag, o);
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, r.key, o);
    r.key = w > r.key ? w : r.key;
  }
  return r;
}

// Row stores (d, per-sample flags) and the band summary of band_rows' result.
template <bool INT>
__device__ __forceinline__ void store_band(const Params& p, int mb, int lane, const BandRows<INT>& r) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int row = mb * BM + lane + 32 * q;
    if (row >= p.M) continue;
    static_cast<unsigned long long*>(p.d)[row] = r.dbits[q];
    p.flags[row] = r.flag[q] ? 1 : 0;
  }
  if (lane == 0) {
    p.ws.band_nflag[mb] = r.nflag;
    p.ws.band_maxkey[mb] = r.key;
  }
}

// The launch summary from the totals.
template <bool INT>
__device__ void publish_summary(const Params& p, int lane, int nf, unsigned long long mk) {
  if (lane == 0) {
    *p.nflag = nf;
    *p.triggered = nf > 0 ? 1 : 0;
    *p.max_disc = (mk == 0ull) ? __longlong_as_double(0x7FF0000000000000ll)
                               : __longlong_as_double(static_cast<long long>(mk - 1ull));
  }
}

// Finished bands' count into the launch summary: atomicMax of their gap key, then an
// acquire-release add of {bands << 32 | flagged rows}; true in the call that completes the count,
// with the launch totals.  (The callers store the band's rows after it: the release then has
// no outstanding stores to wait for.)
__device__ __forceinline__ bool launch_count(const Params& p, int bands, int nflag, unsigned long long key,
                                             unsigned long long& fin_rows, unsigned long long& fin_key) {
  const int total = p.replay ? __ldcg(&p.ws.counters[1]) : p.m_tiles;
  atomicMax(&p.ws.summary[1], key);
  const unsigned long long inc = (static_cast<unsigned long long>(bands) << 32) | static_cast<unsigned>(nflag);
  const unsigned long long old = atom_add_acq_rel_gpu_u64(&p.ws.summary[0], inc);
  if (static_cast<long long>(old >> 32) + bands != total) return false;
  fin_rows = (old + inc) & 0xFFFFFFFFull;
  fin_key = atomicMax(&p.ws.summary[1], 0ull);
  return true;
}

// d / flags of band mb, its band summary and, for the band that completes the launch's
// count, the launch summaries (nflag, triggered, max_disc).  One warp.
template <bool INT>
__device__ void finish_band(const Params& p, int mb, int lane, const unsigned long long (&obs)[4],
                            const unsigned long long (&pred)[4]) {
#ifdef GG_TRACE
  const long long fb_t0 = clock64();
#endif
  const BandRows<INT> r = band_rows<INT>(p, mb, lane, obs, pred);
#ifdef GG_TRACE
  const long long fb_t1 = clock64();
#endif
  int last = 0;
  unsigned long long fin_rows = 0, fin_key = 0;
  if (lane == 0 && !GG_DBG(8192)) last = launch_count(p, 1, r.nflag, r.key, fin_rows, fin_key) ? 1 : 0;
#ifdef GG_TRACE
  const long long fb_t2 = clock64();
#endif
  store_band<INT>(p, mb, lane, r);
#ifdef GG_TRACE
  if (lane == 0 && g_trace != nullptr) {
    const size_t b = static_cast<size_t>(blockIdx.x) * TRACE_TILES * TRACE_EV;
    g_trace[b + 24] = fb_t0;
    g_trace[b + 25] = fb_t1;
    g_trace[b + 26] = fb_t2;
    g_trace[b + 27] = clock64();
  }
#endif
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  publish_summary<INT>(p, lane, static_cast<int>(__shfl_sync(0xffffffffu, fin_rows, 0)),
                       __shfl_sync(0xffffffffu, fin_key, 0));
  if (lane == 0) {
    p.ws.summary[0] = 0ull;  // every band has counted: the workspace is left ready
    p.ws.summary[1] = 0ull;
  }
}

// Error-free fp32 accumulation: (hi, lo) += x with hi + lo exact up to lo's own rounding.
__device__ __forceinline__ void two_sum_acc(float& hi, float& lo, float x) {
  const float t = hi + x, bp = t - hi;
  lo += (hi - (t - bp)) + (x - bp);
  hi = t;
}

// Partial sums travel as 8-byte values (ring slots, workspace partials, reducer
// accumulators): int64 for int8 operands, else an fp32 (hi, lo) double-float pair -- no
// FP64 instruction anywhere in the kernel, whose issue is slow next to the tensor pipe.
enum { ACC_I64 = 0, ACC_DF = 1 };
template <int MODE>
__device__ __forceinline__ unsigned long long acc_add(unsigned long long a, unsigned long long b) {
  if constexpr (MODE == ACC_I64)
    return static_cast<unsigned long long>(static_cast<long long>(a) + static_cast<long long>(b));
  else
    return df_add(a, b);
}

// 16 bytes of the checksum w-vector encoding at byte offset `off`: an explicit
// shared-memory load when the vector was staged there (a generic load would take
// the long L1TEX path), else a read-only global load.
template <bool WSM>
__device__ __forceinline__ uint4 ld_w16(uint32_t w_sm_addr, const void* w_g, int off) {
  if constexpr (WSM) return lds128(w_sm_addr + static_cast<uint32_t>(off));
  else return __ldg(reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(w_g) + off));
}

// One owned K-block of the predicted row sum X[m, kb*BK : (kb+1)*BK] . w (guard.py:168-169)
// from the thread's row copy v (128 bytes, in K order).  w-vectors are zero-padded to
// whole K-blocks (gg_checksum_aux) and TMA zero-fills x beyond K: no tail checks.
template <int KIND, bool WSM>
__device__ __forceinline__ void chk_dot(const uint4 (&v)[8], int kb, uint32_t w_sm_addr, const void* w_g,
                                        float& hi, float& lo, double& accd, long long& acci) {
  if constexpr (KIND == K_I8) {
    // sum_k x*w = sum_d 256^d sum_k x*digit_d(w): exact IDP4A over 128 K per block
    const int base = kb * 512;  // 32 int4 digit triples (+pad) per block
    int a[2][3] = {{0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t x4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 dd = ld_w16<WSM>(w_sm_addr, w_g, base + (j * 4 + q) * 16);
        a[q & 1][0] = __dp4a(static_cast<int>(x4[q]), static_cast<int>(dd.x), a[q & 1][0]);
        a[q & 1][1] = __dp4a(static_cast<int>(x4[q]), static_cast<int>(dd.y), a[q & 1][1]);
        a[q & 1][2] = __dp4a(static_cast<int>(x4[q]), static_cast<int>(dd.z), a[q & 1][2]);
      }
    }
    acci += static_cast<long long>(a[0][0] + a[1][0]) + 256ll * (a[0][1] + a[1][1]) + 65536ll * (a[0][2] + a[1][2]);
  } else if constexpr (KIND == K_TF32) {
    // fp32 x, w = fp32(w_sum): FFMA2 pair chains of 8 products, the block folded into (hi, lo)
    // by TwoSum (no FP64 per element)
    const int base = kb * 32 * 4;  // 32 floats per block
    float2 a[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint4 wq = ld_w16<WSM>(w_sm_addr, w_g, base + j * 16);
      a[0] = fma_f32x2(make_float2(__uint_as_float(v[j].x), __uint_as_float(v[j].y)),
                       make_float2(__uint_as_float(wq.x), __uint_as_float(wq.y)), a[0]);
      a[1] = fma_f32x2(make_float2(__uint_as_float(v[j].z), __uint_as_float(v[j].w)),
                       make_float2(__uint_as_float(wq.z), __uint_as_float(wq.w)), a[1]);
    }
    two_sum_acc(hi, lo, a[0].x);
    two_sum_acc(hi, lo, a[0].y);
    two_sum_acc(hi, lo, a[1].x);
    two_sum_acc(hi, lo, a[1].y);
  } else {
    // bf16/fp16 x is exact in fp32; w = fp32(w_sum) (|w - w_sum| <= 2^-24 |w_sum|).
    // Packed pair FMAs (FFMA2) in two pair chains; bf16 unpacked on the ALU pipe; the
    // block is folded into (hi, lo) by an error-free TwoSum (no FP64 pipe per block).
    const int base = kb * 64 * 4;  // 64 floats per block
    float2 a[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint4 wa = ld_w16<WSM>(w_sm_addr, w_g, base + j * 32);
      const uint4 wb = ld_w16<WSM>(w_sm_addr, w_g, base + j * 32 + 16);
      const float2 wp[4] = {make_float2(__uint_as_float(wa.x), __uint_as_float(wa.y)),
                            make_float2(__uint_as_float(wa.z), __uint_as_float(wa.w)),
                            make_float2(__uint_as_float(wb.x), __uint_as_float(wb.y)),
                            make_float2(__uint_as_float(wb.z), __uint_as_float(wb.w))};
      const uint32_t x4[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 x = (KIND == K_BF16) ? bf16x2_to_f32x2(x4[q])
                                          : __half22float2(*reinterpret_cast<const __half2*>(&x4[q]));
        a[q & 1] = fma_f32x2(x, wp[q], a[q & 1]);
      }
    }
    two_sum_acc(hi, lo, (a[0].x + a[0].y) + (a[1].x + a[1].y));
  }
}

// acc + (one 16-bit half of w) in fp32 with a single mixed-precision add (add.rn.f32.bf16 /
// .f16: FHADD, the half selected by register aliasing); exact conversion, one rounding, so
// the chains equal FADD over the converted values.
template <bool BF16>
__device__ __forceinline__ float add_f32_h16(float acc, uint32_t w, bool high) {
  float r;
  if (high) {
    if constexpr (BF16)
      asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tadd.rn.f32.bf16 %0, h, %2;\n\t}" : "=f"(r) : "r"(w), "f"(acc));
    else
      asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tadd.rn.f32.f16 %0, h, %2;\n\t}" : "=f"(r) : "r"(w), "f"(acc));
  } else {
    if constexpr (BF16)
      asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tadd.rn.f32.bf16 %0, l, %2;\n\t}" : "=f"(r) : "r"(w), "f"(acc));
    else
      asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tadd.rn.f32.f16 %0, l, %2;\n\t}" : "=f"(r) : "r"(w), "f"(acc));
  }
  return r;
}

// Write the 32 output encodings of this thread's box row into the swizzled staging box.
template <int OUT>
__device__ __forceinline__ void stage_row(uint32_t box, int lane, const uint32_t (&o)[32]) {
  if constexpr (OUT == O_I8) {
    const uint32_t row = box + static_cast<uint32_t>(lane * 32);  // SWIZZLE_32B: chunk ^= (row >> 2) & 1
    const int sw = (lane >> 2) & 1;
#pragma unroll
    for (int c = 0; c < 2; ++c)  // o[] holds four bytes per word
      sts128(row + static_cast<uint32_t>((c ^ sw) << 4), o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
  } else if constexpr (OUT == O_BF16 || OUT == O_F16) {
    const uint32_t row = box + static_cast<uint32_t>(lane * 64);  // SWIZZLE_64B: chunk ^= (row >> 1) & 3
    const int sw = (lane >> 1) & 3;
#pragma unroll
    for (int c = 0; c < 4; ++c)  // o[] holds packed pairs
      sts128(row + static_cast<uint32_t>((c ^ sw) << 4), o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
  } else {
    const uint32_t row = box + static_cast<uint32_t>(lane * 128);  // SWIZZLE_128B: chunk ^= row & 7
    const int sw = lane & 7;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      sts128(row + static_cast<uint32_t>((c ^ sw) << 4), o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
  }
}

// Epilogue activations applied to the stored encoding AFTER the observed row sum
// (the check runs on the raw, rounded GEMM output: guard.py:10-11, model.py:367-368,
// SURVEY §8(a) a4 (ii)); the activated value is rounded to the output type again.
enum : int { ACT_NONE = 0, ACT_GELU_TANH = 1, ACT_RELU = 2, ACT_RESIDUAL = 3 };

// model.finish_layer_output's requantisation of an int32 output (model.py:312-316):
// clip(((relu ? max(y, 0) : y) + 2^(s-1)) >> s, -128, 127), int32 wrap-around as NumPy
template <bool RELU>
__device__ __forceinline__ int requant_pre(uint32_t y, int shift) {  // before the saturation
  int h = static_cast<int>(y);
  if constexpr (RELU) h = max(h, 0);
  h = static_cast<int>(static_cast<unsigned>(h) + (1u << (shift - 1)));
  return h >> shift;
}
// four outputs requantised and packed (byte i = output i), saturation by cvt.pack.sat (I2IP)
template <bool RELU>
__device__ __forceinline__ uint32_t requant8x4(const uint32_t* y, int shift) {
  const int a0 = requant_pre<RELU>(y[0], shift), a1 = requant_pre<RELU>(y[1], shift);
  const int a2 = requant_pre<RELU>(y[2], shift), a3 = requant_pre<RELU>(y[3], shift);
  uint32_t hi, w;
  asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(a3), "r"(a2));
  asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(w) : "r"(a1), "r"(a0), "r"(hi));
  return w;
}

// tanh-GELU of an fp32 pair (model._gelu: 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3))));
// tanh on the MUFU pipe (tanh.approx.f32, |rel err| ~2^-11, below bf16 output rounding)
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float2 gelu_tanh_f32x2(float2 x) {
  // u = x (a + b x^2), a = sqrt(2/pi), b = 0.044715 a;  gelu = x (0.5 + 0.5 tanh(u))
  const float2 x2 = mul_f32x2(x, x);
  const float2 p = fma_f32x2(x2, make_float2(0.035677408136300125f, 0.035677408136300125f),
                             make_float2(0.7978845608028654f, 0.7978845608028654f));
  const float2 u = mul_f32x2(x, p);
#ifdef GG_GELU_BF16X2
  // one MUFU for the pair: tanh.approx.bf16x2 on the packed arguments
  uint32_t ub = pack_bf16x2(u.x, u.y), tb;
  asm("tanh.approx.bf16x2 %0, %1;" : "=r"(tb) : "r"(ub));
  const float2 t = bf16x2_to_f32x2(tb);
#else
  const float2 t = make_float2(tanh_approx(u.x), tanh_approx(u.y));
#endif
  return mul_f32x2(x, fma_f32x2(t, make_float2(0.5f, 0.5f), make_float2(0.5f, 0.5f)));
}

template <int KIND, int OUT, bool PROTECT, bool CLAIM, int ACT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    gg_protected_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                                  const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmR,
                                  const Params p) {
  using T = KindTraits<KIND>;
  constexpr bool INT = (KIND == K_I8);
  constexpr int BK = BK_BYTES / T::ELEM;
  constexpr int MMA_K_BYTES = 32;
  constexpr int MMAS_PER_STAGE = BK_BYTES / MMA_K_BYTES;
  constexpr bool OUT16 = (OUT == O_BF16 || OUT == O_F16);
  constexpr bool PRED_PAIR = !INT;  // float kinds: predicted partials as an fp32 (hi, lo) pair
  constexpr int OBS_MODE = INT ? ACC_I64 : ACC_DF;
  constexpr int PRED_MODE = INT ? ACC_I64 : ACC_DF;
  // Split-band folds: claimed in order by every CTA's finisher (CLAIM) or handed to the
  // finisher of the band's last arriver.  The launcher claims for tf32 launches with bands
  // of >= 8 tiles and more than one tile per pair: there a pair that is slightly late is
  // the last arriver of a band in almost every wave, and its finisher backlog (a fold
  // outlasts a tile) made it later still; claiming spreads the folds over all SMs (tf32
  // ViT-B fc1: 30% -> 11% overhead).  A separate instantiation, because compiling the
  // claim loop into a kernel shifts its hot loops' register allocation (128-register cap)
  // and costs every launch of it 4-10 points, claiming or not.
  constexpr bool claim = CLAIM;
  constexpr uint32_t IDESC = PairIdesc<KIND>::V;

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES * A_BYTES;
  uint8_t* smC = smem + C_OFF;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + BAR_OFF);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* aready_bar = empty_bar + STAGES;    // owned stage has landed (relayed by the MMA thread)
  uint64_t* chkdone_bar = aready_bar + STAGES;  // checksum warps copied an owned stage
  uint64_t* tfull_bar = chkdone_bar + STAGES;   // [2]
  uint64_t* tempty_bar = tfull_bar + 2;         // [2] leader: the pair's 8 epilogue warps
  uint64_t* ofull_bar = tempty_bar + 2;         // [NSLOT] observed partials of a tile ready (4 epilogue warps)
  uint64_t* oempty_bar = ofull_bar + NSLOT;     // [NSLOT] consumed by the reducer
  uint64_t* pfull_bar = oempty_bar + NSLOT;     // [NSLOT] predicted partials ready (4 checksum warps)
  uint64_t* pempty_bar = pfull_bar + NSLOT;     // [NSLOT]
  uint64_t* fq_full = pempty_bar + NSLOT;       // [FQ] a split band id queued by the reducer
  uint64_t* fq_empty = fq_full + FQ;            // [FQ] taken by the finisher warp
  uint64_t* rfull_bar = fq_empty + FQ;          // [2 * EPI_WARPS] a residual box landed (TMA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rfull_bar + 2 * EPI_WARPS);
  int* end_fold = reinterpret_cast<int*>(tmem_slot + 1);  // the kernel-end fold: [0] 0 none, 1 every row,
                                                          // 1 + k: the k bands [1], [2]
  int* fq_band = reinterpret_cast<int*>(tmem_slot + 4);           // [FQ]
  double* slot_obs = reinterpret_cast<double*>(tmem_slot + QAREA / 4);  // [NSLOT][2 halves][BM] (int64 bits for INT)
  double* slot_pred = slot_obs + 2 * NSLOT * BM;                // [NSLOT][BM]
  uint32_t* bias_sm = reinterpret_cast<uint32_t*>(slot_pred + NSLOT * BM);  // [2][BN] bias of a tile
  uint8_t* w_sm = reinterpret_cast<uint8_t*>(bias_sm + 2 * BN);              // [W_SMEM] checksum w-vector

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  // predicted row sums computed here from the staged A (the checksum warps), or supplied by
  // the producer of X (p.pred_in: e.g. the layer norm that wrote X), which frees the stages
  const bool own_pred = PROTECT && p.pred_in == nullptr;
  const int n_tiles = p.n_tiles;
  const int m_pairs = (p.M + 2 * BM - 1) / (2 * BM);
  // The pair's tiles: a contiguous range [t0, t1) (bands folded locally) or, when the
  // concurrently streamed A bands would not fit in L2, a strided walk.  A contiguous range
  // is walked as: its leading partial band, its trailing partial band, then its whole bands,
  // so the partial bands' exchange with the neighbouring pairs completes early, off the
  // end of the launch.
  const int pid = static_cast<int>(blockIdx.x >> 1), npairs = static_cast<int>(gridDim.x >> 1);
  int t0, t1;
  pair_range(pid, npairs, m_pairs * n_tiles, t0, t1);
  const int hb = min((t0 + n_tiles - 1) / n_tiles * n_tiles, t1);  // end of the leading partial band
  const int tb = max(t1 / n_tiles * n_tiles, hb);                  // start of the trailing partial band
  // replay: only the listed band pairs (replay_prepare), walked strided
  const int n_walk = p.replay ? __ldcg(&p.ws.counters[2]) * n_tiles : m_pairs * n_tiles;
  const int n_seq = p.sched ? max(0, (n_walk - pid + npairs - 1) / npairs) : t1 - t0;
  auto tile_at = [&](int i) -> int {
    if (p.replay) {
      const int k = pid + i * npairs;
      return __ldcg(&p.ws.active_pairs[k / n_tiles]) * n_tiles + k % n_tiles;
    }
    if (p.sched) return pid + i * npairs;
    if (i < hb - t0) return t0 + i;
    i -= hb - t0;
    if (i < t1 - tb) return tb + i;
    return hb + (i - (t1 - tb));
  };

  // A band pair is folded where it is computed when one pair computes all its N-tiles in
  // order (contiguous schedule, not cut by a range boundary, not a tiny launch): its
  // epilogue and checksum warps keep band totals and hand over once, at the band's last
  // tile.  Other bands hand over every tile and fold through the workspace.  Both paths
  // fold in the same association: per column half, ascending tiles, then the halves.
  auto band_whole = [&](int m) -> bool {
    return !p.sched && !p.tiny && (m * n_tiles >= t0) && ((m + 1) * n_tiles <= t1);
  };

  // band folds shared by the reducer and the finisher warp (protected launches)
  const unsigned long long* so = reinterpret_cast<const unsigned long long*>(slot_obs);
  const unsigned long long* sp = reinterpret_cast<const unsigned long long*>(slot_pred);
  unsigned long long* gpart = reinterpret_cast<unsigned long long*>(p.ws.partial);
  unsigned long long* gpred = reinterpret_cast<unsigned long long*>(p.ws.pred);
  // d / flags of a folded band (one conversion to fp64 per row and band)
  auto finish = [&](int mb, const unsigned long long (&ao)[4], const unsigned long long (&ap)[4]) {
    finish_band<INT>(p, mb, lane, ao, ap);
  };
  // workspace partials of split bands: observed per column half ([half][tile][row]) and predicted
  const size_t half_stride = static_cast<size_t>(n_tiles) * p.m_pad;
  // ascending-tile fold of band b's workspace partials: per half, then the halves (the same
  // association as a band folded where it was computed); FB tiles' loads in flight together
  constexpr int FB = INT ? 2 : 3;  // tiles whose loads are in flight together (register budget)
  auto fold_band = [&](int b, unsigned long long (&bo)[4], unsigned long long (&bpr)[4]) {
    unsigned long long b0[4], b1[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) { b0[q] = 0ull; b1[q] = 0ull; bpr[q] = 0ull; }
    for (int tt0 = 0; tt0 < n_tiles; tt0 += FB) {
      unsigned long long v0[FB][4], v1[FB][4], vp[FB][4];
#pragma unroll
      for (int j = 0; j < FB; ++j) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          v0[j][q] = v1[j][q] = vp[j][q] = 0ull;
          if (tt0 + j < n_tiles) {
            const size_t g = static_cast<size_t>(tt0 + j) * p.m_pad + b * BM + lane + 32 * q;
            v0[j][q] = static_cast<unsigned long long>(ldcg_i64(reinterpret_cast<const long long*>(gpart + g)));
            v1[j][q] = static_cast<unsigned long long>(
                ldcg_i64(reinterpret_cast<const long long*>(gpart + half_stride + g)));
            vp[j][q] = static_cast<unsigned long long>(ldcg_i64(reinterpret_cast<const long long*>(gpred + g)));
          }
        }
      }
#pragma unroll
      for (int j = 0; j < FB; ++j) {
        if (tt0 + j >= n_tiles) break;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          b0[q] = acc_add<OBS_MODE>(b0[q], v0[j][q]);
          b1[q] = acc_add<OBS_MODE>(b1[q], v1[j][q]);
          bpr[q] = acc_add<PRED_MODE>(bpr[q], vp[j][q]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) bo[q] = acc_add<OBS_MODE>(b0[q], b1[q]);
  };
  // warp roles; the SMSP arbiter issues highest-warp-id first, so the ids follow criticality
  constexpr int W_MMA = 15, W_PRODUCER = 14, W_ALLOC = 13, W_REDUCER = 12, W_CHK0 = 8, W_EPI0 = 0;
  if (warp == W_PRODUCER && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (p.c_tma) tma_prefetch(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
      mbar_init(&aready_bar[s], 1);
      mbar_init(&chkdone_bar[s], 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 2 * EPI_WARPS);
    }
    for (int b = 0; b < NSLOT; ++b) {
      mbar_init(&ofull_bar[b], EPI_WARPS);
      mbar_init(&oempty_bar[b], 1);
      mbar_init(&pfull_bar[b], 4);
      mbar_init(&pempty_bar[b], 1);
    }
    for (int b = 0; b < FQ; ++b) {
      mbar_init(&fq_full[b], 1);
      mbar_init(&fq_empty[b], 1);
    }
    for (int b = 0; b < 2 * EPI_WARPS; ++b) {
      mbar_init(&rfull_bar[b], 1);
    }
    end_fold[0] = 0;
    fence_barrier_init();
    fence_proxy_async_smem();
  }
  if (warp == W_ALLOC) {
    tmem_alloc_pair(tmem_slot, TMEM_COLS);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync_all();  // barrier inits and the TMEM allocation visible to both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: the setup above overlapped the previous kernel's tail;
  // nothing below may read memory before that kernel has completed.  The next launch may
  // be scheduled as our CTAs retire.
#ifndef GG_NO_PDL
  pdl_wait();
  pdl_launch_dependents();
#endif

  // replay: a pair tile is recomputed when either of its two 128-row bands is active
  auto pair_active = [&](int m) -> bool {
    if (!p.replay) return true;
    const int b0 = 2 * m, b1 = 2 * m + 1;
    return (b0 < p.m_tiles && p.ws.band_active[b0]) || (b1 < p.m_tiles && p.ws.band_active[b1]);
  };

  if (warp == W_PRODUCER) {
    // ================================================= TMA producer (both CTAs)
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(&full_bar[0]), 0);  // leader's barriers
      int stage = 0;
      uint32_t phase = 0, chk_pending = 0, chk_phase = 0;
#ifdef GG_TRACE
      int plocal = 0;
#endif
      for (int i_seq = 0; i_seq < n_seq; ++i_seq) {
        const int t = tile_at(i_seq);
        const int m = t / n_tiles, n = t - m * n_tiles;
        if (!pair_active(m)) continue;
        const int arow = m * 2 * BM + static_cast<int>(rank) * BM;

        const int brow = n * BN + static_cast<int>(rank) * (BN / 2);
        int rem = 0;  // kb % n_tiles
#ifdef GG_TRACE
        long long tr_empty = 0, tr_chk = 0;
#endif
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          const bool mine = own_pred && rem == n;
          if (++rem == n_tiles) rem = 0;
#ifdef GG_TRACE
          const long long tw0 = clock64();
#endif
          mbar_wait(&empty_bar[stage], phase ^ 1);
#ifdef GG_TRACE
          const long long tw1 = clock64();
          tr_empty += tw1 - tw0;
#endif
          if ((chk_pending & (1u << stage)) && !GG_DBG(2)) {  // the checksum warps still hold the stage's previous K-block
            mbar_wait(&chkdone_bar[stage], (chk_phase >> stage) & 1u);
#ifdef GG_TRACE
            tr_chk += clock64() - tw1;
#endif
            chk_phase ^= 1u << stage;
            chk_pending &= ~(1u << stage);
          }
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * (A_BYTES + B_BYTES));
          const uint32_t fb = full0 + static_cast<uint32_t>(stage * 8);
          tma_load_2d_pair(smA + stage * A_BYTES, &tmA, fb, kb * BK, arow);
          tma_load_2d_pair(smB + stage * B_BYTES, &tmB, fb, kb * BK, brow);
          if (mine) chk_pending |= 1u << stage;
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
#ifdef GG_TRACE
        if (g_trace != nullptr && plocal < TRACE_TILES) {
          const size_t b = (static_cast<size_t>(blockIdx.x) * TRACE_TILES + plocal) * TRACE_EV;
          g_trace[b + 17] = tr_empty;
          g_trace[b + 18] = tr_chk;
        }
        ++plocal;
#endif
      }
    }
  } else if (warp == W_MMA) {
    // ================================================= MMA issuer (leader)
    if (rank == 0 && lane == 0) {
      const uint32_t aready_peer = mapa_shared(smem_u32(&aready_bar[0]), 1);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int i_seq = 0; i_seq < n_seq; ++i_seq) {
        const int t = tile_at(i_seq);
        const int m = t / n_tiles, n = t - m * n_tiles;
        if (!pair_active(m)) continue;
        const int buf = local & 1;
        GG_EV(10, local);
        mbar_wait(&tempty_bar[buf], (static_cast<uint32_t>(local >> 1) & 1u) ^ 1u);
        GG_EV(4, local);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(buf * BN);
#ifdef GG_TRACE
        long long tr_full = 0;
#endif
        int rem = 0;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          const bool mine = own_pred && rem == n;
          if (++rem == n_tiles) rem = 0;
#ifdef GG_TRACE
          const long long tf0 = clock64();
#endif
          mbar_wait(&full_bar[stage], phase);
#ifdef GG_TRACE
          tr_full += clock64() - tf0;
#endif
          if (mine && !GG_DBG(2)) {  // both CTAs' halves of this stage have landed: let the checksum warps copy A
            mbar_arrive(&aready_bar[stage]);
            mbar_arrive_cluster(aready_peer + static_cast<uint32_t>(stage * 8));
          }
          tc_fence_after();
          const uint64_t adesc = sw128_kmajor_desc(smem_u32(smA + stage * A_BYTES));
          const uint64_t bdesc = sw128_kmajor_desc(smem_u32(smB + stage * B_BYTES));
#pragma unroll
          for (int kk = 0; kk < MMAS_PER_STAGE; ++kk)
            tc_mma_pair<T::MMA_KIND>(d_tmem, adesc + static_cast<uint64_t>(kk * (MMA_K_BYTES >> 4)),
                                     bdesc + static_cast<uint64_t>(kk * (MMA_K_BYTES >> 4)), IDESC,
                                     (kb | kk) != 0 ? 1u : 0u);
          tc_commit_pair(&empty_bar[stage], 0x3);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit_pair(&tfull_bar[buf], 0x3);
        GG_EV(5, local);
#ifdef GG_TRACE
        if (g_trace != nullptr && local < TRACE_TILES)
          g_trace[(static_cast<size_t>(blockIdx.x) * TRACE_TILES + local) * TRACE_EV + 19] = tr_full;
#endif
        ++local;
      }
    }
  } else if (warp == W_REDUCER) {
    // ================================================= reducer
    if constexpr (PROTECT) {
      int local = 0, sloti = 0, fq_i = 0;
      for (int i_seq = 0; i_seq < n_seq; ++i_seq) {
        const int t = tile_at(i_seq);
        const int m = t / n_tiles, n = t - m * n_tiles;
        if (!pair_active(m)) continue;
        // band folded where it was computed: one hand-over, at the band's last tile
        const bool whole = band_whole(m);
        if (whole && n != n_tiles - 1) {
          ++local;
          continue;
        }
        const int slot = sloti % NSLOT;
        const uint32_t ph = static_cast<uint32_t>(sloti / NSLOT) & 1u;
        ++sloti;
        if (lane == 0) GG_EV(11, local);
        mbar_wait(&ofull_bar[slot], ph);
        if (lane == 0) GG_EV(12, local);
        mbar_wait(&pfull_bar[slot], ph);
        if (lane == 0) GG_EV(8, local);
        const int mb = 2 * m + static_cast<int>(rank);
        const bool band_ok = mb < p.m_tiles && (!p.replay || p.ws.band_active[mb]) && !GG_DBG(4);
        unsigned long long ao[4], ap[4];
        if (band_ok) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i = lane + 32 * q;
            const int io = 2 * slot * BM + i;  // half 0, then half 1 (+BM)
            const unsigned long long h0 = so[io], h1 = so[io + BM], pv = sp[slot * BM + i];
            if (whole) {  // band totals per half: combine the halves
              ao[q] = acc_add<OBS_MODE>(h0, h1);
              ap[q] = pv;
            } else {      // this tile's partials, per half, into the workspace
              const size_t g = static_cast<size_t>(n) * p.m_pad + mb * BM + i;
              gpart[g] = h0;
              gpart[half_stride + g] = h1;
              gpred[g] = pv;
            }
          }
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&oempty_bar[slot]);
          mbar_arrive(&pempty_bar[slot]);
        }
        if (band_ok) {
          if (whole) {
            if (!GG_DBG(64)) finish(mb, ao, ap);
          } else if ((p.sched || p.tiny || t == min((m + 1) * n_tiles, t1) - 1) && !GG_DBG(128)) {
            // the pair's last tile of this band: release its partials with one count of the
            // tiles it contributed (contiguous schedule: at most two such parts per pair).
            // Tiny launches (at most one tile per pair) count on one launch-wide counter and
            // the CTA of the launch's last tile folds every row with all its threads once its
            // roles are done (after the kernel's closing barrier, below).
            const int part = (p.sched || p.tiny) ? 1 : min((m + 1) * n_tiles, t1) - max(m * n_tiles, t0);
            int* counter = p.tiny ? &p.ws.counters[3] : &p.ws.band_counter[mb];
            __syncwarp();
            int last = 0;
            if (lane == 0) {
#ifdef GG_TRACE
              const long long tt_a = clock64();
#endif
              const int total = p.tiny ? n_tiles * (p.replay ? __ldcg(&p.ws.counters[1]) : p.m_tiles) : n_tiles;
              // acquire-release add: our partials are visible before the count, and the last
              // arriver sees every other pair's partials (no separate fence)
              const int prev = GG_DBG(16) ? atomicAdd(counter, part) : atom_add_acq_rel_gpu(counter, part);
              // claim mode: only a tiny launch's last tile acts; the claimed band's finisher
              // waits for its count to reach n_tiles (one release sequence) and resets it
              last = ((!claim || p.tiny) && prev == total - part) ? 1 : 0;
              if (last) {
                *counter = 0;
                if (p.tiny) end_fold[0] = 1;
#ifdef GG_TRACE
                if (p.tiny && g_trace != nullptr) {
                  const size_t tb0 = static_cast<size_t>(blockIdx.x) * TRACE_TILES * TRACE_EV;
                  g_trace[tb0 + 24] = tt_a;
                  g_trace[tb0 + 25] = clock64();
                }
#endif
              }
            }
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last && !p.tiny && p.few_tiles && !GG_DBG(32)) {
              // at most two tiles per pair: the band is folded at the end of the kernel by all the
              // CTA's threads (at most two such bands per CTA, one per tile)
              if (lane == 0) {
                const int k = end_fold[0] == 0 ? 0 : end_fold[0] - 1;  // bands listed so far
                end_fold[1 + k] = mb;
                end_fold[0] = 2 + k;
              }
            } else if (last && !p.tiny && !GG_DBG(32)) {  // hand the fold to the finisher warp: the reducer keeps draining slots
              if (lane == 0) {
                const int q = fq_i % FQ;
                mbar_wait(&fq_empty[q], (static_cast<uint32_t>(fq_i / FQ) & 1u) ^ 1u);
                fq_band[q] = mb;
                mbar_arrive(&fq_full[q]);
              }
              ++fq_i;
            }
          }
        }
        if (lane == 0) GG_EV(9, local);
        ++local;
      }
      if (lane == 0) {  // end of the finisher's queue
        const int q = fq_i % FQ;
        mbar_wait(&fq_empty[q], (static_cast<uint32_t>(fq_i / FQ) & 1u) ^ 1u);
        fq_band[q] = -1;
        mbar_arrive(&fq_full[q]);
      }
    }
  } else if (warp == W_ALLOC) {
    // ================================================= finisher: folds and finishes split bands
    // handed off by the reducer (acquire ordering: the reducer's fence, then this barrier)
    if constexpr (PROTECT && CLAIM) {
      // Every CTA's finisher claims the launch's split bands in order from one counter and
      // folds each once its count is complete.  Claim lists: strided -- every band;
      // contiguous -- the bands cut by a pair-range boundary; replay -- the active bands.
      if (!p.tiny && !GG_DBG(4) && !GG_DBG(128)) {  // (those diagnostics count no band)
        const int n_claims = p.replay ? 2 * __ldcg(&p.ws.counters[2]) : p.sched ? p.m_tiles : 2 * (npairs - 1);
        for (;;) {
          int idx = 0;
          if (lane == 0) idx = atomicAdd(&p.ws.counters[0], 1);
          idx = __shfl_sync(0xffffffffu, idx, 0);
          if (idx >= n_claims) {  // the launch's last claim leaves the counter ready
            if (lane == 0 && idx == n_claims + static_cast<int>(gridDim.x) - 1) p.ws.counters[0] = 0;
            break;
          }
          int mb;
          if (p.replay) {
            mb = 2 * __ldcg(&p.ws.active_pairs[idx >> 1]) + (idx & 1);
            if (mb >= p.m_tiles || !p.ws.band_active[mb]) continue;
          } else if (p.sched) {
            mb = idx;
          } else {  // the boundary between pairs bp - 1 and bp; one claim per cut band
            int ta, tb, ua, ub;
            const int bp = (idx >> 1) + 1;
            pair_range(bp, npairs, m_pairs * n_tiles, ta, tb);
            if (ta % n_tiles == 0) continue;
            pair_range(bp - 1, npairs, m_pairs * n_tiles, ua, ub);
            if (ua % n_tiles != 0 && ua / n_tiles == ta / n_tiles) continue;
            mb = 2 * (ta / n_tiles) + (idx & 1);
            if (mb >= p.m_tiles) continue;
          }
          if (lane == 0) {  // relaxed polls (no L1 invalidation), then one acquire
            while (ld_relaxed_gpu(&p.ws.band_counter[mb]) != n_tiles) __nanosleep(256);
            fence_acquire_gpu();
          }
          __syncwarp();
          unsigned long long bo[4], bpr[4];
          fold_band(mb, bo, bpr);
          finish(mb, bo, bpr);
          __syncwarp();
          if (lane == 0) p.ws.band_counter[mb] = 0;
        }
      }
    } else if constexpr (PROTECT) {
      for (int i = 0;; ++i) {
        const int q = i % FQ;
        mbar_wait(&fq_full[q], static_cast<uint32_t>(i / FQ) & 1u);
        const int mb = fq_band[q];
        __syncwarp();
        if (lane == 0) mbar_arrive(&fq_empty[q]);
        if (mb < 0) break;
        unsigned long long bo[4], bpr[4];
        fold_band(mb, bo, bpr);
        if (!GG_DBG(256)) finish(mb, bo, bpr);
      }
    }
  } else if (warp >= W_EPI0 && warp < W_EPI0 + EPI_WARPS) {
    // ================================================= epilogue
    const int e = warp - W_EPI0;         // epilogue warp 0..7
    const int eg = warp & 3;             // TMEM lane quadrant (must be warp % 4) / 32-row slab of this CTA
    const int half = e >> 2;             // column half of the tile: chunks 4*half .. 4*half+3
    const int etid = threadIdx.x - 32 * W_EPI0;  // 0..255 over the epilogue warps
    const int tid = eg * 32 + lane;      // accumulator row within this CTA's 128
    const bool lead = (e == 0 && lane == 0);
    const bool c_tma = p.c_tma != 0 && !p.replay;
    const uint32_t tempty0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    int cbuf = 0;
    int local = 0;
    int sloti = 0;                       // hand-overs so far (the reducer's slot sequence)
    unsigned long long band_obs = 0ull;  // whole bands: running total over the band's tiles
    // bias of a tile's 256 columns, one value per epilogue thread, loaded one tile ahead (its
    // latency is off the critical path) and staged in shared memory for the broadcast reads below
    const uint32_t* bias_g = static_cast<const uint32_t*>(p.bias);
    auto bias_of = [&](int i) -> uint32_t {  // bias value of this thread's column in the i-th tile
      if (bias_g == nullptr || i >= n_seq) return 0u;
      const int c = (tile_at(i) % n_tiles) * BN + etid;
      return c < p.N ? __ldcg(bias_g + c) : 0u;
    };
    uint32_t bias_next = bias_of(0);
    // the residual (ACT_RESIDUAL): this thread's row segment of 32 outputs, 16-byte loads
    auto res_load = [&](bool ok, int rrow, int rcol0, uint32_t* dst) {
      if constexpr (ACT == ACT_RESIDUAL && OUT16) {
        const uint16_t* rr = static_cast<const uint16_t*>(p.residual) + static_cast<long long>(rrow) * p.ld_res + rcol0;
        if (ok && rcol0 + 32 <= p.N && (reinterpret_cast<uintptr_t>(rr) & 15) == 0) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(rr) + q);
            dst[4 * q] = u.x; dst[4 * q + 1] = u.y; dst[4 * q + 2] = u.z; dst[4 * q + 3] = u.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const uint32_t lo = ok && rcol0 + 2 * i < p.N ? rr[2 * i] : 0u;
            const uint32_t hi = ok && rcol0 + 2 * i + 1 < p.N ? rr[2 * i + 1] : 0u;
            dst[i] = lo | (hi << 16);
          }
        }
      }
    };
    // the residual through TMA: each epilogue warp's 32 x 32 box loaded into its staging box (the
    // output is then written over it and stored), the next chunk's requested after a store
    const bool r_tma = ACT == ACT_RESIDUAL && OUT16 && p.r_tma != 0 && c_tma;
    uint32_t rph = 0;      // phase bits of this warp's two residual boxes
    bool res_ahead = false;  // the tile's first chunk was requested at the previous tile's last
    auto res_issue = [&](int box_i, int rcol0, int rrow0) {
      uint64_t* bar = &rfull_bar[2 * (warp - W_EPI0) + box_i];
      mbar_arrive_expect_tx(bar, 32 * CBOX * 2);
      tma_load_2d_cta(smC + (warp - W_EPI0) * CST_BYTES + box_i * 2048, &tmR, bar, rcol0, rrow0);
    };
    uint32_t rw_next[ACT == ACT_RESIDUAL ? 16 : 1];
    if constexpr (ACT == ACT_RESIDUAL && OUT16) {
      if (!p.replay && !r_tma && n_seq > 0) {
        const int t2 = tile_at(0);
        const int m2 = t2 / n_tiles, n2 = t2 - m2 * n_tiles;
        const int row2 = m2 * 2 * BM + static_cast<int>(rank) * BM + (warp & 3) * 32 + lane;
        res_load(row2 < p.M, row2, n2 * BN + 32 * (4 * ((warp - W_EPI0) >> 2)), rw_next);
      }
    }
    for (int i_seq = 0; i_seq < n_seq; ++i_seq) {
        const int t = tile_at(i_seq);
      const int m = t / n_tiles, n = t - m * n_tiles;
      if (!pair_active(m)) continue;
      const int buf = local & 1;
      const uint32_t use = static_cast<uint32_t>(local >> 1);
      {
        // bias_next was loaded for tile t unless replay skipped the tiles in between
        const uint32_t bcur = bias_next;
        const int c = n * BN + etid;
        bias_sm[buf * BN + etid] = (p.replay && bias_g != nullptr && c < p.N) ? __ldcg(bias_g + c) : bcur;
        bias_next = bias_of(i_seq + 1);
        named_bar_sync(1, 32 * EPI_WARPS);
      }
      mbar_wait(&tfull_bar[buf], use & 1);
      if (lead) GG_EV(0, local);
      tc_fence_after();
      const int row0 = m * 2 * BM + static_cast<int>(rank) * BM;
      const int row = row0 + tid;
      const bool row_ok = row < p.M;
      const int n0 = n * BN;
      const int nchunks = min(BN / 32, (p.N - n0 + 31) / 32);
      const int c_begin = 4 * half, c_end = min(4 * half + 4, nchunks);
      float obs_hi = 0.f, obs_lo = 0.f;  // float outputs: the tile's observed sum as a double-float
      float obs4[4] = {0.f, 0.f, 0.f, 0.f};  // 16-bit outputs, partial chunks: fp32 chains
      float2 obs_a = make_float2(0.f, 0.f), obs_b = make_float2(0.f, 0.f);  // full chunks: pair chains
      long long obs_i = 0;
      unsigned obs_ilo = 0u;  // int outputs, full chunks: sums of the low / high 16-bit halves
      int obs_ihi = 0;
      int changed = 0;
      // this row's faults: the list is sorted by row (gg_injection), so one binary search per
      // tile finds them and each chunk scans only those (a campaign launch carries one per image)
      int inj_lo = 0, inj_hi = 0;
      if (p.n_inj > 0 && row_ok) {
        int a = 0, b = p.n_inj;
        while (a < b) {
          const int mid = (a + b) >> 1;
          if (p.inj[mid].row < row) a = mid + 1;
          else b = mid;
        }
        inj_lo = a;
        while (b < p.n_inj && p.inj[b].row == row) ++b;
        inj_hi = b;
      }
#ifdef GG_TRACE
      long long tr_ld = 0, tr_cmp = 0, tr_st = 0, tr_obs = 0, tr_t = clock64();
#define GG_LAP(acc)                 \
  do {                              \
    const long long now = clock64(); \
    acc += now - tr_t;              \
    tr_t = now;                     \
  } while (0)
#else
#define GG_LAP(acc) \
  do {              \
  } while (0)
#endif
#pragma unroll 1
      for (int c = c_begin; c < c_end; ++c) {
        const int col0 = n0 + 32 * c;
        // the residual's 32 values of this row and chunk were requested one chunk ahead (their
        // latency overlaps a whole chunk); request the next chunk's -- the next tile's first one
        // after the last (replay walks sparse tiles: loaded here instead)
        uint32_t rw[ACT == ACT_RESIDUAL ? 16 : 1];
        if constexpr (ACT == ACT_RESIDUAL && OUT16) {
          if (r_tma) {
            if (c == c_begin && !res_ahead && lane == 0) {  // a tile's first chunk, not requested ahead
              bulk_wait_read<1>();                          // the box's store two chunks ago has read it
              res_issue(cbuf, col0, row0 + 32 * eg);
            }
            if (c == c_begin) res_ahead = false;
          } else if (p.replay) {
            res_load(row_ok, row, col0, rw);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) rw[i] = rw_next[i];
            if (c + 1 < c_end) {
              res_load(row_ok, row, col0 + 32, rw_next);
            } else if (i_seq + 1 < n_seq) {
              const int t2 = tile_at(i_seq + 1);
              const int m2 = t2 / n_tiles, n2 = t2 - m2 * n_tiles;
              const int row2 = m2 * 2 * BM + static_cast<int>(rank) * BM + tid;
              res_load(row2 < p.M, row2, n2 * BN + 32 * c_begin, rw_next);
            }
          }
        }
        uint32_t r[32];
        tmem_ld_32x32b_x32(
            tmem_base + (static_cast<uint32_t>(eg * 32) << 16) + static_cast<uint32_t>(buf * BN + 32 * c), r);
        tmem_ld_wait();
        GG_LAP(tr_ld);
        if (c == c_end - 1) {  // this warp's TMEM columns drained: tell the leader's MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty0 + static_cast<uint32_t>(buf * 8));
          if (lead) GG_EV(1, local);
        }
        const bool full = (col0 + 32 <= p.N);
        bool out_inj = false;  // an output fault lands in this row's chunk (rare)
        for (int i = inj_lo; i < inj_hi; ++i) {
          const gg_injection f = p.inj[i];
          if (f.col >= col0 && f.col < col0 + 32) {
            if (f.target == GG_INJ_ACCUMULATOR) {
#pragma unroll
              for (int j = 0; j < 32; ++j)  // static indices keep r[] in registers
                if (f.col == col0 + j) r[j] ^= (1u << (f.bit & 31));
            } else {
              out_inj = true;
            }
          }
        }
        // bias (fp32 bits, or int32) of the 32 columns, from the tile's smem copy
        uint32_t bb[32];
        {
          const uint32_t baddr = smem_u32(bias_sm + buf * BN + 32 * c);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint4 bv = lds128(baddr + 16 * q);
            bb[4 * q] = bv.x; bb[4 * q + 1] = bv.y; bb[4 * q + 2] = bv.z; bb[4 * q + 3] = bv.w;
          }
        }
        // o[] holds the stored encodings: packed 16-bit pairs in o[0..15] for bf16/fp16
        // outputs (element 2i in the low half), one 32-bit encoding per column otherwise
        uint32_t o[32];
        if constexpr (OUT16) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {  // packed fp32 pair adds (FADD2), then one cvt per pair
            const float2 v = add_f32x2(make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])),
                                       make_float2(__uint_as_float(bb[2 * i]), __uint_as_float(bb[2 * i + 1])));
            o[i] = (OUT == O_BF16) ? pack_bf16x2(v.x, v.y) : pack_f16x2(v.x, v.y);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = acc_to_out_bits<OUT>(r[j], bb[j]);
        }
        if (out_inj) {
          for (int i = inj_lo; i < inj_hi; ++i) {
            const gg_injection f = p.inj[i];
            if (f.target != GG_INJ_OUTPUT || f.col < col0 || f.col >= col0 + 32) continue;
#pragma unroll
            for (int j = 0; j < 32; ++j) {  // static indices keep o[] in registers
              if (f.col != col0 + j) continue;
              if constexpr (OUT16) {
                const int sh = 16 * (j & 1);
                const uint32_t old = (o[j >> 1] >> sh) & 0xFFFFu;
                const uint32_t nw = (f.mode == GG_INJ_BITFLIP) ? ((old ^ (1u << (f.bit & 31))) & 0xFFFFu)
                                                               : value_to_out_bits<OUT>(f.value);
                o[j >> 1] = (o[j >> 1] & ~(0xFFFFu << sh)) | (nw << sh);
              } else {
                o[j] = (f.mode == GG_INJ_BITFLIP) ? (o[j] ^ (1u << (f.bit & 31))) : value_to_out_bits<OUT>(f.value);
              }
            }
          }
        }
        GG_LAP(tr_cmp);
        if constexpr (PROTECT) {  // observed row sum of the STORED values (guard.py:170)
          if (row_ok && !GG_DBG(8)) {
            if constexpr (INT) {
              if (full) {
                // exact: v = hi16 * 2^16 + lo16 (lo unsigned, hi signed); the halves of two outputs
                // are gathered by PRMT (ALU pipe) and summed by one IDP2A each, into int32 sums that
                // cannot overflow over this thread's <= 128 outputs
#pragma unroll
                for (int j = 0; j < 16; ++j) {  // two outputs per IDP2A: their halves gathered by PRMT
                  const uint32_t lo2 = __byte_perm(o[2 * j], o[2 * j + 1], 0x5410u);
                  const uint32_t hi2 = __byte_perm(o[2 * j], o[2 * j + 1], 0x7632u);
                  obs_ilo = __dp2a_lo(lo2, 0x0101u, obs_ilo);                   // + both lo16 (unsigned)
                  obs_ihi = __dp2a_lo(static_cast<int>(hi2), 0x0101, obs_ihi);  // + both hi16 (signed)
                }
              } else {
                long long s = 0;
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (col0 + j < p.N) s += static_cast<long long>(static_cast<int>(o[j]));
                obs_i += s;
              }
            } else if constexpr (OUT == O_F32) {
              // fp32 outputs: four fp32 chains of 8 (FADD2 pairs), folded per chunk into the
              // double-float (obs_hi, obs_lo) by TwoSum: no FP64 per output
              if (full) {
                float2 c0 = make_float2(0.f, 0.f), c1 = make_float2(0.f, 0.f);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                  const float2 x = make_float2(__uint_as_float(o[2 * i]), __uint_as_float(o[2 * i + 1]));
                  if (i & 1) c1 = add_f32x2(c1, x);
                  else c0 = add_f32x2(c0, x);
                }
                two_sum_acc(obs_hi, obs_lo, c0.x);
                two_sum_acc(obs_hi, obs_lo, c0.y);
                two_sum_acc(obs_hi, obs_lo, c1.x);
                two_sum_acc(obs_hi, obs_lo, c1.y);
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (col0 + j < p.N) two_sum_acc(obs_hi, obs_lo, __uint_as_float(o[j]));
              }
            } else {
              // 16-bit outputs are exact in fp32: four fp32 chains over the tile's 256 columns
              // (error <= 64 * 2^-24 of the chain magnitude, far below the output rounding),
              // folded into fp64 once per tile
              if (full) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {  // mixed-precision adds of the 16-bit halves (FHADD: no
                  // conversion instruction) into four fp32 chains: even pair -> a, odd pair -> b
                  float2& acc = (i & 1) ? obs_b : obs_a;
                  acc.x = add_f32_h16<OUT == O_BF16>(acc.x, o[i], false);
                  acc.y = add_f32_h16<OUT == O_BF16>(acc.y, o[i], true);
                }
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                  const uint32_t h = (o[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
                  if (col0 + j < p.N) obs4[j & 3] += (OUT == O_BF16) ? bf16_bits_to_f32(h) : f16_bits_to_f32(h);
                }
              }
            }
          }
        }
        GG_LAP(tr_obs);
        if constexpr (ACT == ACT_GELU_TANH && OUT16) {  // activation of the checked value, then stored
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 x = (OUT == O_BF16) ? bf16x2_to_f32x2(o[i])
                                             : __half22float2(*reinterpret_cast<const __half2*>(&o[i]));
            const float2 g = gelu_tanh_f32x2(x);
            o[i] = (OUT == O_BF16) ? pack_bf16x2(g.x, g.y) : pack_f16x2(g.x, g.y);
          }
        }
        if constexpr (ACT == ACT_RESIDUAL && OUT16) {
          // the residual stream's update fused: stored = round(residual + y) of the checked y (the
          // bytes a separate add would produce); the residual is read-only here (replayable)
          if (r_tma) {
            mbar_wait(&rfull_bar[2 * (warp - W_EPI0) + cbuf], (rph >> cbuf) & 1u);
            rph ^= 1u << cbuf;
            const uint32_t rrow = smem_u32(smC + (warp - W_EPI0) * CST_BYTES + cbuf * 2048) +
                                  static_cast<uint32_t>(lane * 64);  // SWIZZLE_64B, as stage_row
            const int sw = (lane >> 1) & 3;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint4 u = lds128(rrow + static_cast<uint32_t>((q ^ sw) << 4));
              rw[4 * q] = u.x; rw[4 * q + 1] = u.y; rw[4 * q + 2] = u.z; rw[4 * q + 3] = u.w;
            }
          }
          if (row_ok) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float2 yv = (OUT == O_BF16) ? bf16x2_to_f32x2(o[i])
                                                : __half22float2(*reinterpret_cast<const __half2*>(&o[i]));
              const float2 hv = (OUT == O_BF16) ? bf16x2_to_f32x2(rw[i])
                                                : __half22float2(*reinterpret_cast<const __half2*>(&rw[i]));
              const float2 sv = add_f32x2(hv, yv);
              o[i] = (OUT == O_BF16) ? pack_bf16x2(sv.x, sv.y) : pack_f16x2(sv.x, sv.y);
            }
          }
        }
        if constexpr (OUT == O_I8) {  // the checked int32 outputs requantised, four per word in o[0..7]
          uint32_t h8[8];
#pragma unroll
          for (int v = 0; v < 8; ++v) h8[v] = requant8x4<ACT == ACT_RELU>(o + 4 * v, p.requant_shift);
#pragma unroll
          for (int v = 0; v < 8; ++v) o[v] = h8[v];
        }
        constexpr bool BOX2 = OUT16 || OUT == O_I8;  // boxes of <= 2 KB: two in flight per warp
        if (c_tma) {
          // coalesced store: this warp's 32 rows x 32 columns through a swizzled smem box + TMA
          uint8_t* boxp = smC + e * CST_BYTES + (BOX2 ? cbuf * 2048 : 0);
          if (lane == 0 && !r_tma) {  // (with r_tma the box holds this chunk's residual: already ours)
            if constexpr (BOX2) bulk_wait_read<1>();  // the box written two chunks ago has been read
            else bulk_wait_read<0>();
          }
          __syncwarp();
          stage_row<OUT>(smem_u32(boxp), lane, o);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmC, boxp, col0, row0 + 32 * eg);
            bulk_commit();
          }
          if (r_tma) {  // the next chunk's residual into the other box, once the store two chunks ago
                        // has read it -- at a tile's last chunk, the next tile's first (when it has one)
            int ncol = -1, nrow = 0;
            if (c + 1 < c_end) {
              ncol = col0 + 32;
              nrow = row0 + 32 * eg;
            } else if (i_seq + 1 < n_seq) {
              const int t2 = tile_at(i_seq + 1);
              const int m2 = t2 / n_tiles, n2 = t2 - m2 * n_tiles;
              if (c_begin < min(BN / 32, (p.N - n2 * BN + 31) / 32)) {
                ncol = n2 * BN + 32 * c_begin;
                nrow = m2 * 2 * BM + static_cast<int>(rank) * BM + 32 * eg;
                res_ahead = true;
              }
            }
            if (ncol >= 0 && lane == 0) {
              bulk_wait_read<1>();
              res_issue(cbuf ^ 1, ncol, nrow);
            }
          }
          if constexpr (BOX2) cbuf ^= 1;
          GG_LAP(tr_st);
        } else if (row_ok) {
          if constexpr (OUT == O_I8) {  // 32 requantised bytes of this row per chunk
            const uint32_t* h8 = o;
            uint8_t* cb = static_cast<uint8_t*>(p.C) + static_cast<long long>(row) * p.ldc + col0;
            if (full && (reinterpret_cast<uintptr_t>(cb) & 15) == 0) {
#pragma unroll
              for (int v = 0; v < 2; ++v) {
                uint4* dst = reinterpret_cast<uint4*>(cb) + v;
                if (p.replay) {
                  const uint4 old = *dst;
                  const uint32_t ow[4] = {old.x, old.y, old.z, old.w};
#pragma unroll
                  for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int bq = 0; bq < 4; ++bq) changed += (((ow[q] ^ h8[4 * v + q]) >> (8 * bq)) & 0xFFu) != 0;
                }
                *dst = make_uint4(h8[4 * v], h8[4 * v + 1], h8[4 * v + 2], h8[4 * v + 3]);
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                if (col0 + j >= p.N) continue;
                const uint8_t e = static_cast<uint8_t>(h8[j >> 2] >> (8 * (j & 3)));
                if (p.replay) changed += cb[j] != e ? 1 : 0;
                cb[j] = e;
              }
            }
            continue;
          }
          const long long base = static_cast<long long>(row) * p.ldc + col0;
          constexpr int WORDS = OUT16 ? 16 : 32;  // 32-bit words of this row's 32 outputs
          uint32_t* cw = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(p.C) + base * (OUT16 ? 2 : 4));
          if (full && (reinterpret_cast<uintptr_t>(cw) & 15) == 0) {
            // whole chunk: 16-byte loads / stores; replay counts the outputs whose bytes change
#pragma unroll
            for (int v = 0; v < WORDS / 4; ++v) {
              uint4* dst = reinterpret_cast<uint4*>(cw) + v;
              if (p.replay) {
                const uint4 old = *dst;
                const uint32_t ow[4] = {old.x, old.y, old.z, old.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const uint32_t nw = o[4 * v + q];
                  if constexpr (OUT16)
                    changed += (((ow[q] ^ nw) & 0xFFFFu) != 0) + (((ow[q] ^ nw) >> 16) != 0);
                  else
                    changed += ow[q] != nw;
                }
              }
              *dst = make_uint4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
            }
            continue;
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (col0 + j >= p.N) continue;
            const uint32_t e = OUT16 ? ((o[j >> 1] >> (16 * (j & 1))) & 0xFFFFu) : o[j];
            if (p.replay) changed += (load_out_bits<OUT>(p.C, base + j) != e) ? 1 : 0;
            store_out_bits<OUT>(p.C, base + j, e);
          }
        }
      }
      if (c_begin >= c_end) {  // no columns for this warp in this tile
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty0 + static_cast<uint32_t>(buf * 8));
      }
      if (p.replay && p.changed != nullptr) {
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) changed += __shfl_xor_sync(0xffffffffu, changed, o2);
        if (lane == 0 && changed) atomicAdd(p.changed, changed);
      }
      if constexpr (OUT16) {  // the chains folded exactly into (obs_hi, obs_lo), no FP64 here
        two_sum_acc(obs_hi, obs_lo, obs_a.x);
        two_sum_acc(obs_hi, obs_lo, obs_a.y);
        two_sum_acc(obs_hi, obs_lo, obs_b.x);
        two_sum_acc(obs_hi, obs_lo, obs_b.y);
#pragma unroll
        for (int j = 0; j < 4; ++j) two_sum_acc(obs_hi, obs_lo, obs4[j]);
      }
      if (lead) GG_EV(2, local);
#ifdef GG_TRACE
      if (lead && g_trace != nullptr && local < TRACE_TILES) {
        const size_t b = (static_cast<size_t>(blockIdx.x) * TRACE_TILES + local) * TRACE_EV;
        g_trace[b + 13] = tr_ld;
        g_trace[b + 14] = tr_cmp;
        g_trace[b + 15] = tr_st;
        g_trace[b + 16] = tr_obs;
      }
#endif
      if constexpr (PROTECT) {
        unsigned long long tile_obs;  // this (row, column half)'s partial of the tile, OBS_MODE bits
        if constexpr (INT)
          tile_obs = static_cast<unsigned long long>(obs_i + static_cast<long long>(obs_ihi) * 65536ll +
                                                     static_cast<long long>(obs_ilo));
        else
          tile_obs = static_cast<unsigned long long>(__float_as_uint(obs_hi)) |
                     (static_cast<unsigned long long>(__float_as_uint(obs_lo)) << 32);
        const bool whole = band_whole(m);
        if (whole) band_obs = acc_add<OBS_MODE>(n == 0 ? 0ull : band_obs, tile_obs);
        if (!whole || n == n_tiles - 1) {  // hand over: the tile's partial, or the band's total
          const int slot = sloti % NSLOT;
          mbar_wait(&oempty_bar[slot], (static_cast<uint32_t>(sloti / NSLOT) & 1u) ^ 1u);
          if (lead) GG_EV(3, local);
          reinterpret_cast<unsigned long long*>(slot_obs)[(2 * slot + half) * BM + tid] = whole ? band_obs : tile_obs;
          __syncwarp();
          if (lane == 0) mbar_arrive(&ofull_bar[slot]);
          ++sloti;
        }
      }
      ++local;
    }
    if (c_tma && lane == 0) bulk_wait_all();
  } else if (warp >= W_CHK0 && warp < W_CHK0 + 4) {
    // ================================================= checksum producer side (highest warp ids:
    // the SMSP arbiter issues highest-id-first; these warps are bursty)
    if constexpr (PROTECT) {
      const int cw = warp - W_CHK0;        // rows 32*cw .. 32*cw+31 of this CTA
      const int ctid = threadIdx.x - 32 * W_CHK0;  // 0..127
      const int grp = lane >> 3;           // row within a group of four rows
      const int sub = lane & 7;            // 16-byte piece of a row's 128-byte K-block
      // the whole (zero-padded) w-vector into shared memory once, when it fits
      const bool w_smem = p.w_aux_bytes <= W_SMEM;
      const uint32_t w_sm_addr = smem_u32(w_sm);
      if (w_smem) {
        const uint4* g = static_cast<const uint4*>(p.w_aux);
        uint4* d = reinterpret_cast<uint4*>(w_sm);
        for (int i = ctid; i < p.w_aux_bytes / 16; i += 128) d[i] = __ldg(g + i);
        named_bar_sync(2, 128);
      }
      const int tid = ctid;               // row within this CTA's 128
      const int sw = tid & 7;             // 128B-swizzle phase of this row
      int st0 = 0;                        // pipeline stage of K-block 0 of the current tile
      uint32_t ar_phase = 0;
      // copy this row's 128 B of K-block kb out of its stage and release the stage at once
#ifdef GG_TRACE
      long long tc_wait = 0, tc_copy = 0, tc_fence = 0, tc_comp = 0;
#endif
      auto copy_kb = [&](int kb, uint4 (&v)[8]) {
        const int s = (st0 + kb) % STAGES;
#ifdef GG_TRACE
        const long long c0 = clock64();
#endif
        if (GG_DBG(2)) {
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = make_uint4(kb, s, tid, 0);
          return;
        }
        mbar_wait(&aready_bar[s], (ar_phase >> s) & 1u);  // suspending wait: equal latency, no spin
        ar_phase ^= 1u << s;
#ifdef GG_TRACE
        const long long c1 = clock64();
        tc_wait += c1 - c0;
#endif
        const uint32_t rowaddr = smem_u32(smA + s * A_BYTES) + static_cast<uint32_t>(tid * 128);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = lds128(rowaddr + static_cast<uint32_t>((j ^ sw) << 4));
#ifdef GG_TRACE
        const long long c2 = clock64();
        tc_copy += c2 - c1;
#endif
        // these generic-proxy reads must be ordered before the async-proxy (TMA) refill that the
        // arrive below enables: without the proxy fence the refill can overtake the reads
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&chkdone_bar[s]);
#ifdef GG_TRACE
        tc_fence += clock64() - c2;
#endif
      };
      int local = 0;
      int sloti = 0;                        // hand-overs so far (the reducer's slot sequence)
      unsigned long long band_pred = 0ull;  // whole bands: running total over the band's tiles
      for (int i_seq = 0; i_seq < n_seq; ++i_seq) {
        const int t = tile_at(i_seq);
        const int m = t / n_tiles, n = t - m * n_tiles;
        if (!pair_active(m)) continue;
        double accd = 0.0;
        float hi = 0.f, lo = 0.f;  // bf16/fp16: running block sums, hi + lo exact up to lo's rounding
        long long acci = 0;
        // this tile's share of the band: K-blocks kb == n (mod n_tiles), software-pipelined one
        // deep so an owned stage is released as soon as it lands, not after the previous dot product
        uint4 vc[8], vn[8];
        const int kb0 = own_pred ? n : p.k_blocks;  // supplied predicted sums: no dot products
        if (kb0 < p.k_blocks) copy_kb(kb0, vn);
        for (int kb = kb0; kb < p.k_blocks; kb += n_tiles) {
#pragma unroll
          for (int j = 0; j < 8; ++j) vc[j] = vn[j];
          if (kb + n_tiles < p.k_blocks) copy_kb(kb + n_tiles, vn);
          const uint4 (&v)[8] = vc;
#ifdef GG_TRACE
          const long long cp0 = clock64();
#endif
          if (GG_DBG(1)) { hi += vc[0].x; accd += vc[0].x; acci += vc[1].y; continue; }
          // w-vectors are zero-padded to whole K-blocks (gg_checksum_aux) and TMA zero-fills
          // x beyond K: no tail checks.  Independent accumulators for ILP.
          if (w_smem) chk_dot<KIND, true>(v, kb, w_sm_addr, p.w_aux, hi, lo, accd, acci);
          else chk_dot<KIND, false>(v, kb, w_sm_addr, p.w_aux, hi, lo, accd, acci);
#ifdef GG_TRACE
          // consume the result so the stamp follows the dot product
          if (accd == 1.2345e-300 || acci == 0x7eadbeefll || hi == 1.2345e-30f) tc_comp += 1;
          tc_comp += clock64() - cp0;
#endif
        }
        st0 = (st0 + p.k_blocks) % STAGES;
        if (ctid == 0) GG_EV(6, local);
#ifdef GG_TRACE
        if (ctid == 0 && g_trace != nullptr && local < TRACE_TILES) {
          const size_t b = (static_cast<size_t>(blockIdx.x) * TRACE_TILES + local) * TRACE_EV;
          g_trace[b + 20] = tc_wait;
          g_trace[b + 21] = tc_copy;
          g_trace[b + 22] = tc_fence;
          g_trace[b + 23] = tc_comp;
        }
        tc_wait = tc_copy = tc_fence = tc_comp = 0;
#endif
        unsigned long long tile_pred;  // this row's predicted partial of the tile, PRED_MODE bits
        if (!own_pred) {  // the whole supplied sum enters at the band's tile 0 (folds add zeros elsewhere)
          const long long row = static_cast<long long>(m) * 2 * BM + static_cast<long long>(rank) * BM + tid;
          tile_pred = (n == 0 && row < p.M) ? __ldcg(static_cast<const unsigned long long*>(p.pred_in) + row) : 0ull;
        } else if constexpr (INT) tile_pred = static_cast<unsigned long long>(acci);
        else if constexpr (PRED_PAIR)
          tile_pred = static_cast<unsigned long long>(__float_as_uint(hi)) |
                      (static_cast<unsigned long long>(__float_as_uint(lo)) << 32);
        else tile_pred = static_cast<unsigned long long>(__double_as_longlong(accd));
        const bool whole = band_whole(m);
        if (whole) band_pred = acc_add<PRED_MODE>(n == 0 ? 0ull : band_pred, tile_pred);
        if (!whole || n == n_tiles - 1) {  // hand over: the tile's partial, or the band's total
          const int slot = sloti % NSLOT;
          mbar_wait(&pempty_bar[slot], (static_cast<uint32_t>(sloti / NSLOT) & 1u) ^ 1u);
          if (ctid == 0) GG_EV(7, local);
          reinterpret_cast<unsigned long long*>(slot_pred)[slot * BM + tid] = whole ? band_pred : tile_pred;
          __syncwarp();
          if (lane == 0) mbar_arrive(&pfull_bar[slot]);
          ++sloti;
        }
        ++local;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (PROTECT && !CLAIM) {  // (claim launches have more than two tiles per pair)
    const int ef = end_fold[0];
    if (ef != 0 && !GG_DBG(4096)) {
      // The kernel-end fold, by every thread of the CTA (its roles are done): a tiny launch's
      // last CTA folds every row of the launch (m_tiles * BM <= 512, one per thread); in a
      // launch of at most two tiles per pair, the CTA that completed a band's count folds that
      // band (at most two).
      // Same association as fold_band (per column half over ascending tiles, then the halves).
      // The reducer's acquire-add and the barrier above order the loads.
      const bool every_row = ef == 1;
#ifdef GG_TRACE
      if (every_row && threadIdx.x == 0 && g_trace != nullptr)  // tiny tail: the fold starts
        g_trace[static_cast<size_t>(blockIdx.x) * TRACE_TILES * TRACE_EV + 26] = clock64();
#endif
      const int nb = every_row ? p.m_tiles : ef - 1;  // bands folded here
      const int nrows = nb * BM;
      const int tj = min(static_cast<int>(threadIdx.x) / BM, 1);
      const int r = every_row ? static_cast<int>(threadIdx.x) : end_fold[1 + tj] * BM + static_cast<int>(threadIdx.x) % BM;
      const int b = r / BM;
      int nf = 0;
      unsigned long long key = 0ull, db = 0ull;
      bool fl = false, mine = false;
      if (static_cast<int>(threadIdx.x) < nrows && b < p.m_tiles && (!p.replay || p.ws.band_active[b])) {
        unsigned long long b0 = 0ull, b1 = 0ull, bp = 0ull;
        // four tiles' loads in flight together (measured: 4 beats 2 / 8 / 12 and staging every
        // partial in shared memory first, by cp.async or bulk copies, even at 12 tiles)
        constexpr int TB = 4;
        for (int tt = 0; tt < n_tiles; tt += TB) {
          unsigned long long v0[TB], v1[TB], vp[TB];
#pragma unroll
          for (int j = 0; j < TB; ++j) {
            v0[j] = v1[j] = vp[j] = 0ull;
            if (tt + j < n_tiles) {
              const size_t g = static_cast<size_t>(tt + j) * p.m_pad + r;
              v0[j] = static_cast<unsigned long long>(ldcg_i64(reinterpret_cast<const long long*>(gpart + g)));
              v1[j] = static_cast<unsigned long long>(ldcg_i64(reinterpret_cast<const long long*>(gpart + half_stride + g)));
              vp[j] = static_cast<unsigned long long>(ldcg_i64(reinterpret_cast<const long long*>(gpred + g)));
            }
          }
#pragma unroll
          for (int j = 0; j < TB; ++j) {
            if (tt + j >= n_tiles) break;
            b0 = acc_add<OBS_MODE>(b0, v0[j]);
            b1 = acc_add<OBS_MODE>(b1, v1[j]);
            bp = acc_add<PRED_MODE>(bp, vp[j]);
          }
        }
        if (r < p.M) {
          row_check<INT>(p, acc_add<OBS_MODE>(b0, b1), bp, db, fl, key);
          nf = fl ? 1 : 0;
          mine = true;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        nf += __shfl_xor_sync(0xffffffffu, nf, o);
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, key, o);
        key = w > key ? w : key;
      }
      // per-warp totals in the (idle) observed ring, [16] keys then [16] counts, by explicit
      // shared-space accesses (a generic load here waits behind the warp's global stores)
      const uint32_t red = smem_u32(slot_obs);
      if (lane == 0) {
        sts64(red + 8u * warp, key);
        sts32(red + 128u + 4u * warp, static_cast<uint32_t>(nf));
      }
      __syncthreads();
      if (warp == 0) {
        // lane j: the j-th band folded here (four warps each)
        int bn = 0;
        unsigned long long bk = 0ull;
        if (lane < nb) {
          const int bj = every_row ? lane : end_fold[1 + lane];
          if (p.replay && !p.ws.band_active[bj]) {  // standing summary of an untouched band
            bn = __ldcg(&p.ws.band_nflag[bj]);
            bk = __ldcg(&p.ws.band_maxkey[bj]);
          } else {
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              const int wi = 4 * lane + w;
              bn += static_cast<int>(lds32(red + 128u + 4u * wi));
              const unsigned long long k = lds64(red + 8u * wi);
              bk = k > bk ? k : bk;
            }
            p.ws.band_nflag[bj] = bn;
            p.ws.band_maxkey[bj] = bk;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          bn += __shfl_xor_sync(0xffffffffu, bn, o);
          const unsigned long long w = __shfl_xor_sync(0xffffffffu, bk, o);
          bk = w > bk ? w : bk;
        }
        if (every_row) {
          publish_summary<INT>(p, lane, bn, bk);
#ifdef GG_TRACE
          if (lane == 0 && g_trace != nullptr)  // tiny tail: the summary is out
            g_trace[static_cast<size_t>(blockIdx.x) * TRACE_TILES * TRACE_EV + 27] = clock64();
#endif
        } else {  // the band into the launch count; the band completing it publishes
          int last = 0;
          unsigned long long fin_rows = 0, fin_key = 0;
          if (lane == 0) last = launch_count(p, nb, bn, bk, fin_rows, fin_key) ? 1 : 0;
          last = __shfl_sync(0xffffffffu, last, 0);
          if (last) {
            publish_summary<INT>(p, lane, static_cast<int>(__shfl_sync(0xffffffffu, fin_rows, 0)),
                                 __shfl_sync(0xffffffffu, fin_key, 0));
            if (lane == 0) {
              p.ws.summary[0] = 0ull;  // every band has counted: the workspace is left ready
              p.ws.summary[1] = 0ull;
            }
          }
        }
      }
      if (mine) {  // the rows, after the counts (no outstanding stores for the release to wait on)
        static_cast<unsigned long long*>(p.d)[r] = db;
        p.flags[r] = fl ? 1 : 0;
      }
    }
  }
  cluster_sync_exit();  // the peer's smem / barriers / TMEM stay alive until both CTAs are done
  if (warp == W_ALLOC) tmem_dealloc_pair(tmem_base, TMEM_COLS);
}

}  // namespace pair
}  // namespace gg
