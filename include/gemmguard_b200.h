/*
 * gemmguard_b200.h — C-ABI of the B200-native checksum-protected GEMM path.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `gemmguard` (/root/reference/pkg/src/gemmguard).  The reference has no FFI
 * of its own: its interface is the Python module API.  Each entry point below
 * replaces one reference function (cited file:line); the Python host package
 * `paper_2310_03841_b200` binds them through ctypes and keeps the reference's
 * names, signatures and exceptions.
 *
 * Conventions (all entry points):
 *   - every pointer argument is a DEVICE pointer unless the parameter name
 *     ends in `_host`;
 *   - every call takes a cudaStream_t (passed as void*) and is asynchronous on
 *     it; there are no hidden device synchronisations and no allocations —
 *     the caller owns all memory, including workspace;
 *   - return 0 on success, a negative GG_E* code on failure; the message of
 *     the last failure on the calling thread is `gg_last_error()`;
 *   - re-entrant per stream (workspace must not be shared by concurrent calls).
 */
#ifndef GEMMGUARD_B200_H
#define GEMMGUARD_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GG_API __attribute__((visibility("default")))
#else
#define GG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- element types (reference dtype tags: numerics.py:31-37) ------------ */
enum gg_dtype {
  GG_F64 = 0,   /* "binary64"                                              */
  GG_F32 = 1,   /* "binary32"  (tensor path: kind::tf32)                   */
  GG_F16 = 2,   /* "binary16-emulated" (stored as real fp16 on device)     */
  GG_BF16 = 3,  /* extension: bfloat16 (fields 7,8) — not in the reference */
  GG_I8 = 4,    /* "int8"                                                  */
  GG_I32 = 5,   /* "int32"                                                 */
  GG_I64 = 6,
  GG_TF32X3 = 7 /* operand kind of gg_checksum_aux: fp32 operands run as a
                   3xTF32 split (gg_split_tf32x3), the default for binary32 */
};

/* ---- checksum / accumulation precisions (numerics.py:77-111) ------------ */
enum gg_precision {
  GG_P_F16 = 0, /* Precision.BINARY16  "binary16-emulated" */
  GG_P_F32 = 1, /* Precision.BINARY32  */
  GG_P_F64 = 2, /* Precision.BINARY64  */
  GG_P_I64 = 3  /* Precision.INT64     "int64-exact" */
};

enum gg_statistic { GG_PER_SAMPLE = 0, GG_BATCH_MEAN = 1 };    /* guard.py:93  */
enum gg_inj_target { GG_INJ_OUTPUT = 0, GG_INJ_ACCUMULATOR = 1 };
enum gg_inj_mode { GG_INJ_BITFLIP = 0, GG_INJ_SET_VALUE = 1 }; /* injector.py:49-50 */
/* Epilogue activation applied to each stored output AFTER its observed row sum:
 * the check covers the raw (rounded, bias-included) GEMM output exactly as
 * guard.py:10-11 / model.py:367-368, the activation of that value is what is
 * stored (model.finish_layer_output's GELU, model.py:281-285, 318-319). */
enum gg_epilogue_act { GG_ACT_NONE = 0, GG_ACT_GELU_TANH = 1 /* bf16 / fp16 outputs */,
                       GG_ACT_RELU = 2 /* int8 requantised outputs (c_dtype GG_I8) */,
                       GG_ACT_RESIDUAL = 3 /* bf16 / fp16: C = residual + y (desc.residual) */ };

enum gg_error {
  GG_OK = 0,
  GG_EINVAL = -1,     /* bad argument (shape, dtype, alignment, domain)   */
  GG_ECUDA = -2,      /* CUDA runtime / driver failure                    */
  GG_EWORKSPACE = -3, /* workspace too small                              */
  GG_EUNSUPPORTED = -4
};

/* One fault to inject inside the protected GEMM epilogue.
 * target OUTPUT flips bit `bit` of the stored encoding of C[row, col] (or
 * replaces it by `value` rounded to the output type) after bias add and
 * rounding, before the observed checksum — injector.py:265-271 /
 * guard.py:515-523.  target ACCUMULATOR flips the raw fp32/s32 TMEM
 * accumulator before the bias add (build extension).
 * An injection list must be sorted by row (ascending; ties in any order):
 * each epilogue thread binary-searches it once per tile. */
typedef struct gg_injection {
  int64_t row;
  int32_t col;
  int32_t bit;
  int32_t target; /* gg_inj_target */
  int32_t mode;   /* gg_inj_mode   */
  double value;   /* used when mode == GG_INJ_SET_VALUE */
} gg_injection;

/* Descriptor of one protected GEMM launch:
 *     C[m, n] = sum_k A[m, k] * B[n, k] + bias[n]
 * A is the layer input X [M, K] row-major; B is the weight in torch layout
 * W [N, K] row-major (K-major), i.e. the transpose of the reference's stored
 * Wt [K, N] (model.py:43).  With protect=1 the epilogue also produces the
 * per-row discrepancy d[m] = (sum_k A[m,k]*w_sum[k] + bias_sum) - sum_n C[m,n]
 * over the STORED (rounded, bias-included, possibly injected) outputs, the
 * flags and the summary scalars of guard._verify_arrays (guard.py:188-215). */
typedef struct gg_gemm_desc {
  int32_t ab_kind;  /* GG_BF16 | GG_F16 | GG_F32 (tf32 MMA) | GG_I8       */
  int32_t c_dtype;  /* float kinds: GG_BF16 | GG_F16 | GG_F32; GG_I8: GG_I32 */
  int64_t M, N, K;
  const void* A; int64_t lda; /* elements; lda*size % 16 == 0, A 16B aligned */
  const void* B; int64_t ldb; /* elements; ldb*size % 16 == 0, B 16B aligned */
  const void* bias;           /* [N] f32 (float kinds) or i32 (GG_I8); NULL = 0 */
  void* C; int64_t ldc;       /* elements */

  int32_t protect;            /* 0: unprotected baseline of the same kernel  */
  int32_t chk_prec;           /* GG_P_F64 / F32 / F16 (float kinds: d is formed in
                                 double-float and reported in binary64 for all
                                 three, at least the reference's precision) or
                                 GG_P_I64 (GG_I8)                               */
  const void* w_sum;          /* [K] f64 or i64: gg_offline_checksum output  */
  const void* w_aux;          /* gg_checksum_aux output for this ab_kind     */
  double bias_sum_f;          /* bias_sum for GG_P_F64                       */
  int64_t bias_sum_i;         /* bias_sum for GG_P_I64                       */
  double mu, lo, hi;          /* EpsilonModel mu, threshold_low/high         */
  int32_t statistic;          /* gg_statistic                                */

  void* d;                    /* [M] f64 (GG_P_F64) or i64 (GG_P_I64)        */
  uint8_t* flags;             /* [M] 0/1                                     */
  double* max_disc;           /* scalar                                      */
  int32_t* nflag;             /* scalar: number of flagged rows              */
  uint8_t* triggered;         /* scalar 0/1                                  */

  const gg_injection* inj;    /* device array sorted by row, may be NULL     */
  int32_t n_inj;

  void* workspace;            /* zero-filled before first use; every call    */
  size_t workspace_bytes;     /* leaves it zero-filled again on completion   */

  /* replay (gg_replay_tiles only): */
  const uint8_t* replay_rows; /* [M] rows whose M-bands are recomputed       */
  int32_t* changed;           /* scalar: outputs whose bytes changed         */

  int32_t epilogue_act;       /* gg_epilogue_act (0: store the GEMM output)   */

  /* Optional predicted row sums PRED[m] = sum_k A[m,k] * w_sum[k] computed by
   * the producer of A (e.g. gg_add_layernorm's pred_out for the layer it
   * feeds) as fp32 (hi, lo) pairs, hi in the low word; NULL: K1 forms them
   * from its staged A tiles.  Float kinds only.  With it the kernel's
   * checksum warps do no dot products and hold no pipeline stage. */
  const void* pred_in;

  /* Layout of B: GG_B_NK (0) = [N, K] row-major (torch Linear, K-major: what the
   * tensor cores read) or GG_B_KN (1) = [K, N] row-major (the reference's Wt,
   * model.py:43; ldb >= N).  With GG_B_KN the launcher first transposes B into
   * b_scratch (caller-owned device memory of gg_b_scratch_bytes(ab_kind, N, K)
   * bytes) on the stream; callers that reuse a weight should transpose it once. */
  int32_t b_layout;
  void* b_scratch;
  size_t b_scratch_bytes;

  /* Int8 operands with c_dtype = GG_I8: the stored output is the requantised hidden state
   * h = clip(((relu ? max(y, 0) : y) + 2^(s-1)) >> s, -128, 127) of the int32 GEMM output y
   * (int32 wrap-around, arithmetic shift: model.finish_layer_output's requantisation,
   * model.py:312-316), s = requant_shift in [1, 30], relu with epilogue_act = GG_ACT_RELU.
   * The check runs on y (guard.py:170: the GEMM output, before the layer glue); C is [M, N]
   * int8 (ldc in bytes). */
  int32_t requant_shift;

  /* epilogue_act = GG_ACT_RESIDUAL (16-bit outputs): the stored output is the residual
   * stream's update round(residual + y) of the checked GEMM output y (the check covers y,
   * guard.py:170; the add is a transformer block's glue).  residual [M, N] (ld_res, the
   * output type) must not alias C, so a replay can recompute the same bytes. */
  const void* residual;
  int64_t ld_res;
} gg_gemm_desc;

enum gg_b_layout { GG_B_NK = 0, GG_B_KN = 1 };

/* Bytes of b_scratch a GG_B_KN launch needs: N rows of K elements padded to 16 bytes. */
GG_API size_t gg_b_scratch_bytes(int32_t ab_kind, int64_t N, int64_t K);

/* Library identity. */
GG_API const char* gg_last_error(void);
GG_API int gg_version(void);

/* Bytes of workspace gg_protected_gemm / gg_replay_tiles need for (M, N). */
GG_API size_t gg_protected_gemm_workspace_bytes(int64_t M, int64_t N);

/* K1 — protected GEMM (tcgen05 + TMEM + TMA, sm_100a).
 * Replaces numerics.gemm (numerics.py:237-289) + model.run_layer
 * (model.py:334-338) + guard._discrepancies (guard.py:163-171) +
 * guard._verify_arrays (guard.py:188-215) fused in one launch.
 * Float kinds: both sides of d accumulate as fp32 (hi, lo) pairs in fixed
 * orders, and d = (pred + bias_sum_f) - obs is rounded once to binary64 (no FP64
 * instruction runs in the kernel); |d - fp64 d| <= 2^-19 * sum of |terms|, and
 * repeated launches and replays give bit-identical d.  Int8: d is exact int64. */
GG_API int gg_protected_gemm(const gg_gemm_desc* desc, void* stream);

/* K4 — replay only the M-bands holding a row with replay_rows[m] != 0, with
 * the identical tile configuration and K order as gg_protected_gemm, writing
 * the recomputed tiles into C, counting outputs whose bytes changed into
 * *changed, and re-deriving d/flags/summaries over all rows.
 * Replaces guard._replay (guard.py:575-604). */
GG_API int gg_replay_tiles(const gg_gemm_desc* desc, void* stream);

/* Tile localisation by column checksums (north_star kernel (1): e^T A and the
 * column sums of C; not in the reference, which checks rows only, SPEC.md:497,
 * and replays the whole layer, guard.py:575-604).  For every 128-row band
 * holding a row with flags[r] != 0, the column discrepancies
 *   e[b, n] = (sum_{r in b} X[r, :]) . W[n, :] + rows_b * bias[n] - sum_{r in b} C[r, n]
 * (int64 for int8 operands, fp64 otherwise) and tile_mask[b * n_tiles + t] = 1
 * for each 256-column tile t holding a column with e != 0 (int8), or (floats)
 * a non-finite e or |e| > frac * min over the band's flagged rows with a
 * finite d of |d[r] - mu|.
 * X [M, K] (ldx) and W [N, K] (ldw, torch layout) of x_dtype (GG_BF16, GG_F16,
 * GG_F32, GG_I8); C [M, N] (ldc) of c_dtype (the K1 output type); bias [N] of
 * bias_dtype or NULL; d the K1 result's d (f64, or i64 for int8).  tile_mask:
 * ceil(M/128) x ceil(N/256) bytes (zeroed here); col_disc (optional, may be
 * NULL): ceil(M/128) x N values, written for the flagged bands only.
 * workspace: gg_locate_workspace_bytes(M, K) bytes of device scratch. */
GG_API size_t gg_locate_workspace_bytes(int64_t M, int64_t K);
GG_API int gg_locate_tiles(int32_t x_dtype, const void* X, int64_t M, int64_t K, int64_t ldx,
                           const void* W, int64_t N, int64_t ldw, const void* bias,
                           int32_t bias_dtype, int32_t c_dtype, const void* C, int64_t ldc,
                           const uint8_t* flags, const void* d, double mu, double frac,
                           uint8_t* tile_mask, void* col_disc, void* workspace,
                           size_t workspace_bytes, void* stream);

/* K2 — offline weight checksum w_sum[k] = sum_n W[n,k] (ascending n) and
 * bias_sum = sum_n bias[n] in precision chk_prec; bit-exact with
 * guard.offline_checksum (guard.py:142-160, _accumulate_in 135-139).
 * w_layout 0: W is [N, K] row-major (torch); 1: W is Wt [K, N] (reference).
 * w_sum_out: [K] of the precision's type (f16/f32/f64/i64);
 * bias_sum_out: one element of that type.  bias may be NULL (sum = 0). */
GG_API int gg_offline_checksum(int32_t w_dtype, const void* W, int64_t K, int64_t N,
                        int64_t ldw, int32_t w_layout, const void* bias,
                        int32_t bias_dtype, int32_t chk_prec, void* w_sum_out,
                        void* bias_sum_out, void* stream);

/* Side-path encoding of w_sum consumed by the fused checksum of K1, computed
 * once per weight (offline, like w_sum itself), zero-padded to a multiple of
 * 128 K-elements so the kernel reads whole K-blocks:
 *   GG_BF16 / GG_F16: float [Kp]  = fp32(w_sum); bf16/fp16 x are exact in fp32,
 *                     so x*w is one fp32 FMA (|w - w_sum| <= 2^-24 |w_sum|),
 *                     folded by TwoSum into an fp32 (hi, lo) pair;
 *   GG_F32 (tf32):    float  [Kp] = fp32(w_sum) (as the 16-bit kinds);
 *   GG_TF32X3:        float [3*Ks, padded to 128] = [0 | w | w] over the
 *                     three segments of a gg_split_tf32x3 expansion (K is the
 *                     original K; Ks = K rounded up to 32);
 *   GG_I8:            int32x4 [Kp/4] signed base-256 digit planes of the int64
 *                     w_sum (|w_sum| < 2^23), so x*w_sum is an exact IDP4A dot. */
GG_API size_t gg_checksum_aux_bytes(int32_t ab_kind, int64_t K);
GG_API int gg_checksum_aux(int32_t ab_kind, const void* w_sum, int64_t K, void* aux_out,
                           void* stream);

/* binary32 at binary32 accuracy on the tf32 tensor pipe (3xTF32).  Expands an
 * fp32 operand [rows, K] (row pitch ld) into dst [rows, 3*Ks] (row pitch ldd >=
 * 3*Ks, Ks = K rounded up to 32; pads zero):
 *   role 0 (A = X): [hi | lo | hi]        role 1 (B = W [N, K]): [lo | hi | hi]
 * with hi = x rounded to tf32 (RNE) and lo = x - hi (exact in fp32).  A
 * gg_protected_gemm launch with ab_kind GG_F32 over the expanded operands
 * (K' = 3*Ks) accumulates hi*lo + lo*hi + hi*hi per product in fp32 — the
 * binary32 product of numerics.gemm (numerics.py:222-234) to ~2^-21 instead of
 * tf32's 2^-11, small cross terms first because the tensor core's fp32
 * accumulator truncates each step by a fraction of its own magnitude — and,
 * with w_aux = gg_checksum_aux(GG_TF32X3, w_sum, K), its predicted row sum is
 * (lo + hi) . w = x . w exactly as before.  Non-finite x are kept whole in the
 * last segment (zeros elsewhere).  Plain single-pass TF32 stays available as
 * an explicit opt-in (ab_kind GG_F32 on x itself). */
GG_API int gg_split_tf32x3(const float* src, int64_t rows, int64_t K, int64_t ld, int32_t role,
                           float* dst, int64_t ldd, void* stream);

/* Reference-exact verification of a given (X, Y): sequential folds in the
 * checksum precision exactly as guard._discrepancies (guard.py:163-171) and
 * the flag/summary rules of guard._verify_arrays (guard.py:188-215).
 * X [M, K] (ldx) of x_dtype, Y [M, N] (ldy) of y_dtype, w_sum [K] and
 * bias_sum (one element) of the precision's type.  d_out is f64 for float
 * precisions and i64 for GG_P_I64.  max_disc/nflag/triggered as above. */
GG_API int gg_verify_rows(int32_t x_dtype, const void* X, int64_t M, int64_t K,
                   int64_t ldx, int32_t y_dtype, const void* Y, int64_t N,
                   int64_t ldy, int32_t chk_prec, const void* w_sum,
                   const void* bias_sum, double mu, double lo, double hi,
                   int32_t statistic, void* d_out, uint8_t* flags_out,
                   double* max_disc_out, int32_t* nflag_out,
                   uint8_t* triggered_out, void* stream);

/* K3 — flip bit bit_idx[i] of element elem_idx[i] of the buffer `ptr` whose
 * elements are elem_bytes wide (1, 2, 4 or 8), for i < n (device arrays).
 * The flip is an involution: call twice to restore.  Replaces
 * numerics.flip_bit (numerics.py:308-321) for operand/weight locations. */
GG_API int gg_flip_bits(void* ptr, int32_t elem_bytes, const int64_t* elem_idx,
                 const int32_t* bit_idx, int64_t n, void* stream);

/* Reference-exact GEMM on CUDA cores: ascending-k single accumulator in the
 * accumulation precision, products rounded before the add, result rounded to
 * the operand dtype — bit-exact with numerics.gemm (numerics.py:222-289)
 * for every (dtype, accum) pair the reference accepts.  Used for parity and
 * as the binary64 path; the tensor path is gg_protected_gemm.
 * X [M, K] row-major, Wt [K, N] row-major (reference layout), bias [N] of
 * the accumulation type (or i32 for integers), Y [M, N] of the operand type
 * (i32 for integer operands). */
GG_API int gg_gemm_exact(int32_t dtype, int32_t accum, const void* X, int64_t M,
                  int64_t K, const void* Wt, int64_t N, const void* bias,
                  void* Y, void* stream);

/* numerics.reduce_rows / reduce_cols (numerics.py:292-305): ascending f64
 * (i64 for integer dtypes) folds; axis 1 = per row, axis 0 = per column. */
GG_API int gg_reduce(int32_t dtype, const void* A, int64_t rows, int64_t cols,
              int32_t axis, void* out, void* stream);

/* Elementwise helpers used by the host package (all device arrays). */
GG_API int gg_round_f64_to(int32_t dtype, const double* in, void* out, int64_t n,
                    void* stream); /* RNE: numerics._round_array 202-208 */

/* Calibration statistics (guard.calibrate_epsilon, guard.py:300-355): merge
 * the n discrepancies d[0..n) (f64, device) into the device-resident running
 * state[3] = {count, mean, M2} (Welford per chunk, Chan's pairwise merge over
 * a fixed tree: deterministic).  sigma = sqrt(M2 / (count - 1)). Zero the
 * state before the first batch. */
GG_API int gg_running_stats(const double* d, int64_t n, double* state, void* stream);

/* Range profiling (profiler.profile_ranges, profiler.py:62-80): update the
 * running state[3] = {key(min), key(max), non-finite count} with the finite
 * values of Y [M, N] (row pitch ldy elements; dtype GG_BF16, GG_F16, GG_F32 or
 * GG_I32).  key(v) maps a double onto uint64 preserving order: bits | 2^63
 * for v >= 0, ~bits for v < 0.  Initialise state to {~0, 0, 0}. */
GG_API int gg_minmax(int32_t dtype, const void* Y, int64_t M, int64_t N, int64_t ldy,
                     uint64_t* state, void* stream);

/* Integer toy-pipeline glue (model.finish_layer_output for integer models,
 * model.py:307-331), batched: Y [B*T, N] int32 raw GEMM outputs (row pitch ldy)
 * -> H int8 hidden state.  relu (mlp_fc1) then requantise
 * clip((h + 2^(shift-1)) >> shift, -128, 127); for qkv layers (qkv != 0) also
 * the head mix floor((q+k+v)/3) and token mix floor((m + floor(sum_t m / T)) / 2)
 * per sample, giving H [B*T, N/3].  NumPy integer semantics: bit-exact. */
GG_API int gg_int_finish(const int32_t* Y, int64_t B, int64_t T, int64_t N, int64_t ldy,
                         int32_t relu, int32_t shift, int32_t qkv, int8_t* H, void* stream);

/* Transformer glue of the protected ViT / Swin forward (not a reference
 * function: the reference's toy pipeline glue is model.prepare_layer_input /
 * finish_layer_output, model.py:288-331; attention and layer norm stay
 * unprotected as in PAPER.md:221).  Residual update and layer norm in one
 * pass: if y != NULL, h_out = round(h + y) (h_out may alias h); then
 * ln_out = LN(h_out or h) * gamma + beta with fp32 statistics over rows of D
 * (D a multiple of 32 x 16 bytes up to 8 such chunks per lane; dtype
 * GG_BF16, GG_F16 or GG_F32; 16-byte aligned, contiguous rows).  ln_out must
 * not alias h, y or h_out (GG_EINVAL). */
GG_API int gg_add_layernorm(int32_t dtype, const void* h, const void* y, int64_t rows, int64_t D,
                            const float* gamma, const float* beta, float eps, void* h_out,
                            void* ln_out, const float* w_pred, uint64_t* pred_out, void* stream);
/* ViT patch extraction: images [B, C, H, W] (NCHW) -> the patch-embedding GEMM's
 * input [B * (H/P) * (W/P), C * P * P], row (b, gy, gx), column (c, py, px); 16-byte
 * copies (P * element size a multiple of 16 bytes, 16-byte aligned tensors). */
GG_API int gg_patchify(int32_t dtype, const void* images, int64_t B, int64_t C, int64_t H, int64_t W,
                       int64_t P, void* out, void* stream);
/* The ViT embedding's tail in one pass: the residual stream h_out [B*T, D] is
 * row (b, 0) = cls + pos[0] and row (b, t) = e[b*(T-1) + t-1] + pos[t] (t >= 1),
 * each sum rounded to dtype like torch's add (e: the patch-embedding GEMM's
 * output [B*(T-1), D], pos [T, D], cls [D]), then ln_out = LN(h_out) * gamma +
 * beta as gg_add_layernorm (w_pred / pred_out likewise). */
GG_API int gg_embed_layernorm(int32_t dtype, const void* e, const void* pos, const void* cls, int64_t B,
                              int64_t T, int64_t D, const float* gamma, const float* beta, float eps,
                              void* h_out, void* ln_out, const float* w_pred, uint64_t* pred_out,
                              void* stream);
/* If w_pred != NULL (the consumer layer's gg_checksum_aux vector, fp32 w_sum),
 * also pred_out[row] = sum_k ln_out[row,k] * w_pred[k] over the STORED (rounded)
 * ln_out values, as an fp32 (hi, lo) pair with lo = 0 (a per-lane fp32 FMA chain
 * and a fixed butterfly over the warp: error <= (D/32 + 5) 2^-24 sum |x w|,
 * inside the fused check's 2^-19 sum |terms| bound): the pred_in of the
 * protected GEMM that consumes ln_out (guard.py:168-169's predicted side). */

#ifdef __cplusplus
}
#endif
#endif /* GEMMGUARD_B200_H */
