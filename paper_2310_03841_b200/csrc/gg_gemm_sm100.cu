// gg_gemm_sm100.cu — host launcher of K1 (protected GEMM) and K4 (replay).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <string>

#include "gg_gemm2_sm100.cuh"
#include "gg_internal.h"

namespace gg {

namespace {

unsigned long long f64_bits_host(double x) {
  unsigned long long b;
  std::memcpy(&b, &x, sizeof b);
  return b;
}

// x as an fp32 (hi, lo) pair, hi in the low word (the kernels' double-float format)
unsigned long long df_split(double x) {
  const float h = static_cast<float>(x);
  const float l = std::isfinite(h) ? static_cast<float>(x - static_cast<double>(h)) : 0.0f;
  uint32_t uh, ul;
  std::memcpy(&uh, &h, sizeof uh);
  std::memcpy(&ul, &l, sizeof ul);
  return static_cast<unsigned long long>(uh) | (static_cast<unsigned long long>(ul) << 32);
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D K-major operand [rows, K] with row pitch ld_bytes; box = (128 B of K, box_rows).
int make_operand_map(CUtensorMap* map, CUtensorMapDataType dt, int elem, const void* ptr, int64_t K, int64_t rows,
                     int64_t ld_bytes, uint32_t box_rows) {
  auto enc = tensor_map_encoder();
  if (enc == nullptr) return fail(GG_ECUDA, "cuTensorMapEncodeTiled is unavailable (driver too old?)");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_bytes)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(pair::BK_BYTES / elem), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(GG_ECUDA, "cuTensorMapEncodeTiled failed (code " + std::to_string(int(r)) + ")");
  return 0;
}

// Output map for the TMA-store epilogue: [M, N] row-major with pitch ld_bytes,
// box = 32 columns x 32 rows, swizzle matching the epilogue's smem staging.
int make_output_map(CUtensorMap* map, CUtensorMapDataType dt, int elem, void* ptr, int64_t N, int64_t M,
                    int64_t ld_bytes) {
  auto enc = tensor_map_encoder();
  if (enc == nullptr) return fail(GG_ECUDA, "cuTensorMapEncodeTiled is unavailable (driver too old?)");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(M)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_bytes)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(pair::CBOX), static_cast<cuuint32_t>(pair::CBOX)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, dt, 2, ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   elem == 1 ? CU_TENSOR_MAP_SWIZZLE_32B : elem == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(GG_ECUDA, "cuTensorMapEncodeTiled (C) failed (code " + std::to_string(int(r)) + ")");
  return 0;
}

int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  static int cache[64] = {0};
  if (dev >= 0 && dev < 64 && cache[dev]) return cache[dev];
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cache[dev] = n;
  return n;
}

struct WsLayout {
  size_t summary, counters, band_counter, band_active, active_pairs, band_nflag, band_maxkey, pred, partial, total;
};
inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
WsLayout ws_layout(int64_t M, int64_t N) {
  const size_t m_tiles = static_cast<size_t>((M + BM - 1) / BM);
  const size_t n_tiles = static_cast<size_t>((N + BN - 1) / BN);
  const size_t m_pad = m_tiles * BM;
  WsLayout L{};
  size_t off = 0;
  L.summary = off; off += 16;
  L.counters = off; off = align_up(off + 16, 256);
  L.band_counter = off; off = align_up(off + 4 * m_tiles, 256);
  L.band_active = off; off = align_up(off + m_tiles, 256);
  L.active_pairs = off; off = align_up(off + 4 * ((m_tiles + 1) / 2), 256);
  L.band_nflag = off; off = align_up(off + 4 * m_tiles, 256);
  L.band_maxkey = off; off = align_up(off + 8 * m_tiles, 256);
  L.pred = off; off = align_up(off + 8 * m_pad * n_tiles, 256);
  L.partial = off; off = align_up(off + 2 * 8 * m_pad * n_tiles, 256);  // per column half
  L.total = off;
  return L;
}

// Replay: mark the 128-row bands holding flagged rows and seed the launch summary with the
// inactive bands' standing summaries (the replayed bands add theirs); with no active band
// the summary is final here.
__global__ void replay_prepare_kernel(const uint8_t* rows, int M, int m_tiles, uint8_t* band_active, int* counters,
                                      int* active_pairs,
                                      unsigned long long* summary, const int* band_nflag,
                                      const unsigned long long* band_maxkey, int* changed, int* nflag,
                                      uint8_t* triggered, double* max_disc) {
  __shared__ int s_count, s_rows;
  __shared__ unsigned long long s_key;
  if (threadIdx.x == 0) {
    s_count = 0;
    s_rows = 0;
    s_key = 0ull;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int m = warp; m < m_tiles; m += nw) {
    int any = 0;
    for (int r = m * BM + lane; r < min((m + 1) * BM, M); r += 32) any |= rows[r] ? 1 : 0;
    any = __any_sync(0xffffffffu, any);
    if (lane == 0) {
      band_active[m] = any ? 1 : 0;
      if (any) {
        atomicAdd(&s_count, 1);
      } else {
        atomicAdd(&s_rows, band_nflag[m]);
        atomicMax(&s_key, band_maxkey[m]);
      }
    }
  }
  __syncthreads();
  // ascending list of the 256-row band pairs holding an active band (block-wide scan)
  __shared__ int s_off[1024];
  const int m_pairs = (m_tiles + 1) / 2;
  const int per = (m_pairs + blockDim.x - 1) / blockDim.x;
  const int p0 = min(m_pairs, static_cast<int>(threadIdx.x) * per), p1 = min(m_pairs, p0 + per);
  int mine = 0;
  for (int q = p0; q < p1; ++q) mine += (band_active[2 * q] || (2 * q + 1 < m_tiles && band_active[2 * q + 1])) ? 1 : 0;
  s_off[threadIdx.x] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int i = 0; i < static_cast<int>(blockDim.x); ++i) {
      const int c = s_off[i];
      s_off[i] = acc;
      acc += c;
    }
    counters[2] = acc;
  }
  __syncthreads();
  int at = s_off[threadIdx.x];
  for (int q = p0; q < p1; ++q)
    if (band_active[2 * q] || (2 * q + 1 < m_tiles && band_active[2 * q + 1])) active_pairs[at++] = q;
  if (threadIdx.x == 0) {
    counters[1] = s_count;
    if (changed) *changed = 0;
    if (s_count > 0) {
      summary[0] = static_cast<unsigned long long>(static_cast<unsigned>(s_rows));
      summary[1] = s_key;
    } else {
      *nflag = s_rows;
      *triggered = s_rows > 0 ? 1 : 0;
      *max_disc = (s_key == 0ull) ? __longlong_as_double(0x7FF0000000000000ll)
                                  : __longlong_as_double(static_cast<long long>(s_key - 1ull));
    }
  }
}

// Per device, once per instantiation: the shared-memory opt-in is a per-device
// function attribute (a process driving several GPUs configures each one).
template <int KIND, int OUT, bool PROTECT, bool CLAIM, int ACT>
int configure_instance(int dev) {
  static std::mutex mu;
  static bool done[64] = {false};
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return 0;
  auto kern = pair::gg_protected_gemm_pair_kernel<KIND, OUT, PROTECT, CLAIM, ACT>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pair::SMEM_BYTES) != cudaSuccess)
    return fail(GG_ECUDA, "cudaFuncSetAttribute(max dynamic smem, pair kernel) failed");
  done[dev] = true;
  return 0;
}

int current_device(int& dev) {
  dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return fail(GG_EUNSUPPORTED, "protected_gemm: device ordinal beyond 63");
  return 0;
}

// CTA pairs that can be resident at once on this device (every instantiation has the
// same shared memory and block size).  The grid never exceeds it: the claimed split-band
// folds (CLAIM) spin on bands owned by other pairs, so a pair that could not be
// scheduled (MPS limits, green contexts, kernels on other streams) would hang the launch.
int max_coresident_pairs(int dev) {
  static std::mutex mu;
  static int cache[64] = {0};
  std::lock_guard<std::mutex> lk(mu);
  if (cache[dev]) return cache[dev];
  auto kern = pair::gg_protected_gemm_pair_kernel<K_BF16, O_BF16, true, false, pair::ACT_NONE>;
  int n = 0;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pair::SMEM_BYTES) == cudaSuccess) {
    cudaLaunchConfig_t occ{};
    occ.gridDim = dim3(2);
    occ.blockDim = dim3(pair::THREADS);
    occ.dynamicSmemBytes = pair::SMEM_BYTES;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &occ) != cudaSuccess) n = 0;
  }
  cudaGetLastError();
  if (n < 1) n = num_sms() / 2;
  cache[dev] = n;
  return n;
}

template <int KIND, int OUT, bool PROTECT, bool CLAIM = false, int ACT = pair::ACT_NONE>
int launch_pair_instance(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const CUtensorMap& tr,
                         const Params& p, int grid, cudaStream_t s) {
  auto kern = pair::gg_protected_gemm_pair_kernel<KIND, OUT, PROTECT, CLAIM, ACT>;
  int dev;
  int rc = current_device(dev);
  if (rc) return rc;
  rc = configure_instance<KIND, OUT, PROTECT, CLAIM, ACT>(dev);
  if (rc) return rc;
#ifdef GG_NO_PDL
  kern<<<grid, pair::THREADS, pair::SMEM_BYTES, s>>>(ta, tb, tc, tr, p);
#else
  // programmatic dependent launch: the CTA setup overlaps the previous kernel's tail (the
  // kernel waits on griddepcontrol before touching memory)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(pair::THREADS);
  cfg.dynamicSmemBytes = pair::SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, tr, p);
#endif
  return check_launch("protected_gemm_pair");
}

template <int KIND, int OUT>
int dispatch_protect(bool protect, int act, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                     const CUtensorMap& tr, const Params& p, int grid, cudaStream_t s) {
  if constexpr ((KIND == K_BF16 && OUT == O_BF16) || (KIND == K_F16 && OUT == O_F16)) {
    if (act == GG_ACT_GELU_TANH)
      return protect ? launch_pair_instance<KIND, OUT, true, false, pair::ACT_GELU_TANH>(ta, tb, tc, tr, p, grid, s)
                     : launch_pair_instance<KIND, OUT, false, false, pair::ACT_GELU_TANH>(ta, tb, tc, tr, p, grid, s);
    if (act == GG_ACT_RESIDUAL)
      return protect ? launch_pair_instance<KIND, OUT, true, false, pair::ACT_RESIDUAL>(ta, tb, tc, tr, p, grid, s)
                     : launch_pair_instance<KIND, OUT, false, false, pair::ACT_RESIDUAL>(ta, tb, tc, tr, p, grid, s);
  }
  if constexpr (OUT == O_I8) {
    if (act == GG_ACT_RELU)
      return protect ? launch_pair_instance<KIND, OUT, true, false, pair::ACT_RELU>(ta, tb, tc, tr, p, grid, s)
                     : launch_pair_instance<KIND, OUT, false, false, pair::ACT_RELU>(ta, tb, tc, tr, p, grid, s);
  }
  if (act != GG_ACT_NONE)
    return fail(GG_EUNSUPPORTED,
                "protected_gemm: GELU / residual need bf16 / fp16 outputs, ReLU requantised int8 outputs");
  if (!protect) return launch_pair_instance<KIND, OUT, false>(ta, tb, tc, tr, p, grid, s);
  if constexpr (KIND == K_TF32) {  // claimed split-band folds (see the kernel)
    if (!p.few_tiles && !p.tiny && p.n_tiles >= 8) return launch_pair_instance<KIND, OUT, true, true>(ta, tb, tc, tr, p, grid, s);
  }
  return launch_pair_instance<KIND, OUT, true>(ta, tb, tc, tr, p, grid, s);
}

}  // namespace

size_t protected_gemm_workspace_bytes(int64_t M, int64_t N) { return ws_layout(M, N).total; }

namespace {
// [K, N] (ld = ldb) -> [N, Kp] row-major through 32 x 32 shared tiles (coalesced both sides)
template <typename E>
__global__ void transpose_kn_kernel(const E* __restrict__ src, int64_t K, int64_t N, int64_t ldb, E* __restrict__ dst,
                                    int64_t ldd) {
  __shared__ E tile[32][33];
  const int64_t k0 = static_cast<int64_t>(blockIdx.y) * 32, n0 = static_cast<int64_t>(blockIdx.x) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t k = k0 + i, n = n0 + threadIdx.x;
    if (k < K && n < N) tile[i][threadIdx.x] = src[k * ldb + n];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t n = n0 + i, k = k0 + threadIdx.x;
    if (n < N && k < K) dst[n * ldd + k] = tile[threadIdx.x][i];
  }
}

int64_t padded_k(int elem, int64_t K) {
  const int64_t step = 16 / elem;
  return (K + step - 1) / step * step;
}
}  // namespace

size_t b_scratch_bytes(int ab_kind, int64_t N, int64_t K) {
  const int elem = ab_kind == GG_F32 ? 4 : ab_kind == GG_I8 ? 1 : 2;
  return static_cast<size_t>(N) * static_cast<size_t>(padded_k(elem, K)) * static_cast<size_t>(elem);
}

int launch_protected_gemm(const gg_gemm_desc* d, bool replay, cudaStream_t s) {
  if (d == nullptr) return fail(GG_EINVAL, "protected_gemm: null descriptor");
  if (d->b_layout == GG_B_KN) {
    // the reference's Wt [K, N]: transposed into the caller's scratch, then the K-major launch
    const int elem = d->ab_kind == GG_F32 ? 4 : d->ab_kind == GG_I8 ? 1 : 2;
    if (d->ab_kind != GG_BF16 && d->ab_kind != GG_F16 && d->ab_kind != GG_F32 && d->ab_kind != GG_I8)
      return fail(GG_EUNSUPPORTED, "protected_gemm: ab_kind must be GG_BF16, GG_F16, GG_F32 or GG_I8");
    if (d->N < 1 || d->K < 1) return fail(GG_EINVAL, "gemm dims mismatch: M, N, K must be positive");
    if (d->B == nullptr || d->b_scratch == nullptr) return fail(GG_EINVAL, "protected_gemm: GG_B_KN needs B and b_scratch");
    if (d->ldb < d->N) return fail(GG_EINVAL, "protected_gemm: GG_B_KN needs ldb >= N");
    if (d->b_scratch_bytes < b_scratch_bytes(d->ab_kind, d->N, d->K))
      return fail(GG_EWORKSPACE, "protected_gemm: b_scratch too small (gg_b_scratch_bytes)");
    if (reinterpret_cast<uintptr_t>(d->b_scratch) & 15) return fail(GG_EINVAL, "protected_gemm: b_scratch must be 16-byte aligned");
    const int64_t kp = padded_k(elem, d->K);
    const dim3 grid(static_cast<unsigned>((d->N + 31) / 32), static_cast<unsigned>((d->K + 31) / 32)), block(32, 8);
    if (grid.y > 65535) return fail(GG_EUNSUPPORTED, "protected_gemm: GG_B_KN with K beyond 2^21");
    switch (elem) {
      case 1: transpose_kn_kernel<uint8_t><<<grid, block, 0, s>>>(static_cast<const uint8_t*>(d->B), d->K, d->N, d->ldb,
                                                                  static_cast<uint8_t*>(d->b_scratch), kp); break;
      case 2: transpose_kn_kernel<uint16_t><<<grid, block, 0, s>>>(static_cast<const uint16_t*>(d->B), d->K, d->N, d->ldb,
                                                                   static_cast<uint16_t*>(d->b_scratch), kp); break;
      default: transpose_kn_kernel<uint32_t><<<grid, block, 0, s>>>(static_cast<const uint32_t*>(d->B), d->K, d->N, d->ldb,
                                                                    static_cast<uint32_t*>(d->b_scratch), kp); break;
    }
    if (const int rc = check_launch("protected_gemm (B transpose)")) return rc;
    gg_gemm_desc nk = *d;
    nk.B = d->b_scratch;
    nk.ldb = kp;
    nk.b_layout = GG_B_NK;
    return launch_protected_gemm(&nk, replay, s);
  }
  if (d->b_layout != GG_B_NK) return fail(GG_EINVAL, "protected_gemm: b_layout must be GG_B_NK or GG_B_KN");
  if (d->M < 1 || d->N < 1 || d->K < 1) return fail(GG_EINVAL, "gemm dims mismatch: M, N, K must be positive");
  if (d->M > (int64_t(1) << 30) || d->N > (int64_t(1) << 30) || d->K > (int64_t(1) << 30))
    return fail(GG_EINVAL, "protected_gemm: dims beyond 2^30");
  int kind, elem;
  CUtensorMapDataType tdt;
  switch (d->ab_kind) {
    case GG_BF16: kind = K_BF16; elem = 2; tdt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16; break;
    case GG_F16: kind = K_F16; elem = 2; tdt = CU_TENSOR_MAP_DATA_TYPE_FLOAT16; break;
    case GG_F32: kind = K_TF32; elem = 4; tdt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32; break;
    case GG_I8: kind = K_I8; elem = 1; tdt = CU_TENSOR_MAP_DATA_TYPE_UINT8; break;
    default: return fail(GG_EUNSUPPORTED, "protected_gemm: ab_kind must be GG_BF16, GG_F16, GG_F32 or GG_I8");
  }
  int out;
  switch (d->c_dtype) {
    case GG_BF16: out = O_BF16; break;
    case GG_F16: out = O_F16; break;
    case GG_F32: out = O_F32; break;
    case GG_I32: out = O_I32; break;
    case GG_I8: out = O_I8; break;
    default: return fail(GG_EUNSUPPORTED, "protected_gemm: unsupported c_dtype");
  }
  const bool int_kind = kind == K_I8;
  if (int_kind != (out == O_I32 || out == O_I8))
    return fail(GG_EINVAL, "protected_gemm: int8 operands produce int32 (or requantised int8) outputs only");
  if (out == O_I8 && (d->requant_shift < 1 || d->requant_shift > 30))
    return fail(GG_EINVAL, "protected_gemm: int8 outputs need a requant shift in [1, 30]");
  if (kind == K_BF16 && out == O_F16) return fail(GG_EUNSUPPORTED, "protected_gemm: bf16 -> f16 output not built");
  if (kind == K_F16 && out == O_BF16) return fail(GG_EUNSUPPORTED, "protected_gemm: f16 -> bf16 output not built");
  if (kind == K_TF32 && out != O_F32) return fail(GG_EUNSUPPORTED, "protected_gemm: tf32 produces f32 outputs only");
  if ((reinterpret_cast<uintptr_t>(d->A) & 15) || (reinterpret_cast<uintptr_t>(d->B) & 15))
    return fail(GG_EINVAL, "protected_gemm: A and B must be 16-byte aligned");
  if ((d->lda * elem) % 16 || (d->ldb * elem) % 16)
    return fail(GG_EINVAL, "protected_gemm: lda/ldb must be multiples of 16 bytes");
  if (d->lda < d->K || d->ldb < d->K || d->ldc < d->N) return fail(GG_EINVAL, "protected_gemm: leading dims too small");
  const bool protect = d->protect != 0;
  if (protect || replay) {
    if (int_kind && d->chk_prec != GG_P_I64)
      return fail(GG_EINVAL, "integer layers require the int64-exact checksum precision");
    // float kinds: d is formed in double-float and rounded once to binary64 whatever the
    // requested checksum precision (binary16 / binary32 / binary64): at least as precise as the
    // reference's folds in that precision (guard.py:135-139), never less
    if (!int_kind && d->chk_prec != GG_P_F64 && d->chk_prec != GG_P_F32 && d->chk_prec != GG_P_F16)
      return fail(GG_EINVAL, "float layers take a floating checksum precision");
    if (reinterpret_cast<uintptr_t>(d->w_sum) & 15) return fail(GG_EINVAL, "protected_gemm: w_sum must be 16-byte aligned");
    if (d->w_aux == nullptr || (reinterpret_cast<uintptr_t>(d->w_aux) & 15))
      return fail(GG_EINVAL, "protected_gemm: w_aux (gg_checksum_aux) is required and must be 16-byte aligned");
    if (!d->w_sum || !d->d || !d->flags || !d->max_disc || !d->nflag || !d->triggered)
      return fail(GG_EINVAL, "protected_gemm: protect=1 needs w_sum, d, flags, max_disc, nflag, triggered");
    if (!d->workspace || d->workspace_bytes < protected_gemm_workspace_bytes(d->M, d->N))
      return fail(GG_EWORKSPACE, "protected_gemm: workspace too small");
  }
  if (replay && !protect) return fail(GG_EINVAL, "replay_tiles: requires protect=1");
  if (int_kind && protect && d->N > 65535)
    return fail(GG_EUNSUPPORTED, "protected_gemm: int8 checksum path supports N <= 65535 (|w_sum| < 2^23)");
  if (int_kind && protect && d->K > (int64_t(1) << 17))
    return fail(GG_EUNSUPPORTED, "protected_gemm: int8 checksum path supports K <= 131072");
  if (replay && d->replay_rows == nullptr) return fail(GG_EINVAL, "replay_tiles: replay_rows is NULL");
  if (d->n_inj < 0 || (d->n_inj > 0 && d->inj == nullptr)) return fail(GG_EINVAL, "protected_gemm: bad injection list");

  CUtensorMap ta, tb;
  int rc = make_operand_map(&ta, tdt, elem, d->A, d->K, d->M, d->lda * elem, BM);
  if (rc) return rc;
  rc = make_operand_map(&tb, tdt, elem, d->B, d->K, d->N, d->ldb * elem, pair::BN / 2);
  if (rc) return rc;
  // C through the TMA-store epilogue when the pointer and pitch allow it
  const int out_elem = (out == O_BF16 || out == O_F16) ? 2 : out == O_I8 ? 1 : 4;
  const CUtensorMapDataType cdt = out == O_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                  : out == O_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                  : out == O_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                  : out == O_I8  ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                                 : CU_TENSOR_MAP_DATA_TYPE_INT32;
  CUtensorMap tc;
  std::memset(&tc, 0, sizeof(tc));
  int c_tma = ((reinterpret_cast<uintptr_t>(d->C) & 15) == 0 && (d->ldc * out_elem) % 16 == 0) ? 1 : 0;
  if (c_tma && make_output_map(&tc, cdt, out_elem, d->C, d->N, d->M, d->ldc * out_elem) != 0) c_tma = 0;
  // the fused residual update's input, through the same 32 x 32 boxes as the stores
  CUtensorMap tr = tc;
  int r_tma = 0;
  if (d->epilogue_act == GG_ACT_RESIDUAL && c_tma && d->residual != nullptr &&
      (reinterpret_cast<uintptr_t>(d->residual) & 15) == 0 && (d->ld_res * out_elem) % 16 == 0 &&
      make_output_map(&tr, cdt, out_elem, const_cast<void*>(d->residual), d->N, d->M, d->ld_res * out_elem) == 0)
    r_tma = 1;

  Params p{};
  p.M = static_cast<int>(d->M);
  p.N = static_cast<int>(d->N);
  p.K = static_cast<int>(d->K);
  p.m_tiles = static_cast<int>((d->M + BM - 1) / BM);
  p.n_tiles = static_cast<int>((d->N + BN - 1) / BN);
  p.k_blocks = static_cast<int>((d->K * elem + pair::BK_BYTES - 1) / pair::BK_BYTES);
  p.m_pad = p.m_tiles * BM;
  p.A = d->A;
  p.lda = d->lda;
  p.C = d->C;
  p.ldc = d->ldc;
  p.c_tma = c_tma;
  p.requant_shift = d->requant_shift;
  if (d->epilogue_act == GG_ACT_RESIDUAL) {
    if (d->residual == nullptr || d->ld_res < d->N)
      return fail(GG_EINVAL, "protected_gemm: GG_ACT_RESIDUAL needs the residual [M, N] (ld_res >= N)");
    if (d->residual == d->C) return fail(GG_EINVAL, "protected_gemm: the residual must not alias C (replay reads it)");
  }
  p.residual = d->residual;
  p.ld_res = d->ld_res;
  p.r_tma = r_tma;
#ifdef GG_DIAGNOSTICS
  if (std::getenv("GG_NO_CTMA")) p.c_tma = 0;  // diagnostics: direct vector stores from registers
#endif
  {
    static const int dbg = [] {
      const char* e = std::getenv("GG_DEBUG");
      return e ? std::atoi(e) : 0;
    }();
    p.dbg = dbg;
  }
  p.bias = d->bias;
  p.w_sum = d->w_sum;
  p.w_aux = d->w_aux;
  p.w_aux_bytes = static_cast<int>(checksum_aux_bytes(d->ab_kind, d->K));
  p.bias_sum_f = d->bias_sum_f;
  p.bias_sum_i = d->bias_sum_i;
  p.mu = d->mu;
  p.lo = d->lo;
  p.hi = d->hi;
  p.bias_df = df_split(d->bias_sum_f);
  p.neg_mu_df = df_split(-d->mu);
  p.mu_zero = d->mu == 0.0 ? 1 : 0;
  p.lo_key = std::isnan(d->lo) ? ~0ull : f64_order_key(f64_bits_host(d->lo));  // NaN bounds: every row flags
  p.hi_key = std::isnan(d->hi) ? 0ull : f64_order_key(f64_bits_host(d->hi));
  // the kernel applies the per-sample rule; batch_mean flags need every d and are
  // re-derived below by one pairwise-mean pass (guard.py:198-201)
  const bool batch_mean = !int_kind && protect && d->statistic == GG_BATCH_MEAN;
  p.statistic = GG_PER_SAMPLE;
  p.d = d->d;
  p.flags = d->flags;
  p.max_disc = d->max_disc;
  p.nflag = d->nflag;
  p.triggered = d->triggered;
  p.inj = d->inj;
  p.n_inj = d->n_inj;
  p.replay = replay ? 1 : 0;
  p.pred_in = d->pred_in;
  if (d->pred_in != nullptr) {
    if (int_kind) return fail(GG_EUNSUPPORTED, "protected_gemm: pred_in is for float kinds (fp32 pair sums)");
    if (reinterpret_cast<uintptr_t>(d->pred_in) & 7) return fail(GG_EINVAL, "protected_gemm: pred_in must be 8-byte aligned");
  }

  p.changed = d->changed;
  if (protect) {
    const WsLayout L = ws_layout(d->M, d->N);
    uint8_t* w = static_cast<uint8_t*>(d->workspace);
    p.ws.summary = reinterpret_cast<unsigned long long*>(w + L.summary);
    p.ws.counters = reinterpret_cast<int*>(w + L.counters);
    p.ws.band_counter = reinterpret_cast<int*>(w + L.band_counter);
    p.ws.band_active = w + L.band_active;
    p.ws.active_pairs = reinterpret_cast<int*>(w + L.active_pairs);
    p.ws.band_nflag = reinterpret_cast<int*>(w + L.band_nflag);
    p.ws.band_maxkey = reinterpret_cast<unsigned long long*>(w + L.band_maxkey);
    p.ws.pred = reinterpret_cast<double*>(w + L.pred);
    p.ws.partial = reinterpret_cast<double*>(w + L.partial);
  }
  if (replay) {
    replay_prepare_kernel<<<1, 1024, 0, s>>>(d->replay_rows, p.M, p.m_tiles, p.ws.band_active, p.ws.counters,
                                              p.ws.active_pairs, p.ws.summary, p.ws.band_nflag, p.ws.band_maxkey, d->changed,
                                              d->nflag, d->triggered, d->max_disc);
    rc = check_launch("replay_prepare");
    if (rc) return rc;
  }
  int dev;
  rc = current_device(dev);
  if (rc) return rc;
  const int pair_tiles = ((p.M + 2 * pair::BM - 1) / (2 * pair::BM)) * p.n_tiles;
  const int pairs = std::min(pair_tiles, std::min(num_sms() / 2, max_coresident_pairs(dev)));
  const int grid = 2 * pairs;
  // A bands streamed concurrently by all pairs (256 rows x K each): keep them L2-resident
  const double a_footprint = static_cast<double>(pairs) * 2 * pair::BM * static_cast<double>(d->K) * elem;
  p.sched = a_footprint > 40.0e6 ? 1 : 0;
#ifdef GG_DIAGNOSTICS
  if (p.dbg & 1024) p.sched = 0;  // diagnostics: force a schedule
  if (p.dbg & 2048) p.sched = 1;
#endif
  if (replay) p.sched = 1;  // replay walks the listed band pairs strided; every band folds via the workspace
  // tiny launches (at most one tile per pair, <= 4 bands): one launch-wide count, every row
  // folded by the threads of the last arriving CTA
  p.tiny = (pair_tiles <= pairs && p.m_tiles <= 4) ? 1 : 0;  // one fold thread per row (<= 512)
  p.few_tiles = (pair_tiles <= 2 * pairs && !replay) ? 1 : 0;

  switch (kind) {
    case K_BF16:
      rc = out == O_BF16 ? dispatch_protect<K_BF16, O_BF16>(protect, d->epilogue_act, ta, tb, tc, tr, p, grid, s)
                         : dispatch_protect<K_BF16, O_F32>(protect, d->epilogue_act, ta, tb, tc, tr, p, grid, s);
      break;
    case K_F16:
      rc = out == O_F16 ? dispatch_protect<K_F16, O_F16>(protect, d->epilogue_act, ta, tb, tc, tr, p, grid, s)
                        : dispatch_protect<K_F16, O_F32>(protect, d->epilogue_act, ta, tb, tc, tr, p, grid, s);
      break;
    case K_TF32:
      rc = dispatch_protect<K_TF32, O_F32>(protect, d->epilogue_act, ta, tb, tc, tr, p, grid, s);
      break;
    default:
      rc = out == O_I32 ? dispatch_protect<K_I8, O_I32>(protect, d->epilogue_act, ta, tb, tc, tr, p, grid, s)
                        : dispatch_protect<K_I8, O_I8>(protect, d->epilogue_act, ta, tb, tc, tr, p, grid, s);
  }
  if (rc == 0 && batch_mean)
    rc = launch_batch_mean_finish(d->M, d->mu, d->lo, d->hi, static_cast<const double*>(d->d), d->flags, d->max_disc,
                                  d->nflag, d->triggered, s);
  return rc;
}

#ifdef GG_TRACE
extern "C" __attribute__((visibility("default"))) int gg_trace_buffer(void* buf) {
  unsigned long long* b = static_cast<unsigned long long*>(buf);
  return cudaMemcpyToSymbol(pair::g_trace, &b, sizeof(b)) == cudaSuccess ? 0 : GG_ECUDA;
}
#endif

}  // namespace gg
