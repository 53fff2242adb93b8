// gg_capi.cu — extern "C" entry points declared in include/gemmguard_b200.h.
// Plain pointers and sizes only; no torch types cross this boundary.
#include <cuda_runtime.h>

#include <string>

#include "gg_internal.h"

namespace gg {

namespace {
thread_local std::string g_last_error;
}

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(GG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return 0;
}

}  // namespace gg

extern "C" {

const char* gg_last_error(void) { return gg::g_last_error.c_str(); }

int gg_version(void) { return 10000; }  // 1.0.0

size_t gg_protected_gemm_workspace_bytes(int64_t M, int64_t N) {
  if (M < 1 || N < 1) return 0;
  return gg::protected_gemm_workspace_bytes(M, N);
}

int gg_protected_gemm(const gg_gemm_desc* desc, void* stream) {
  return gg::launch_protected_gemm(desc, false, static_cast<cudaStream_t>(stream));
}

int gg_replay_tiles(const gg_gemm_desc* desc, void* stream) {
  return gg::launch_protected_gemm(desc, true, static_cast<cudaStream_t>(stream));
}

size_t gg_checksum_aux_bytes(int32_t ab_kind, int64_t K) { return gg::checksum_aux_bytes(ab_kind, K); }

int gg_checksum_aux(int32_t ab_kind, const void* w_sum, int64_t K, void* aux_out, void* stream) {
  return gg::launch_checksum_aux(ab_kind, w_sum, K, aux_out, static_cast<cudaStream_t>(stream));
}

int gg_split_tf32x3(const float* src, int64_t rows, int64_t K, int64_t ld, int32_t role, float* dst, int64_t ldd,
                    void* stream) {
  return gg::launch_split_tf32x3(src, rows, K, ld, role, dst, ldd, static_cast<cudaStream_t>(stream));
}

int gg_offline_checksum(int32_t w_dtype, const void* W, int64_t K, int64_t N, int64_t ldw, int32_t w_layout,
                        const void* bias, int32_t bias_dtype, int32_t chk_prec, void* w_sum_out,
                        void* bias_sum_out, void* stream) {
  return gg::launch_offline_checksum(w_dtype, W, K, N, ldw, w_layout, bias, bias_dtype, chk_prec, w_sum_out,
                                     bias_sum_out, static_cast<cudaStream_t>(stream));
}

int gg_verify_rows(int32_t x_dtype, const void* X, int64_t M, int64_t K, int64_t ldx, int32_t y_dtype, const void* Y,
                   int64_t N, int64_t ldy, int32_t chk_prec, const void* w_sum, const void* bias_sum, double mu,
                   double lo, double hi, int32_t statistic, void* d_out, uint8_t* flags_out, double* max_disc_out,
                   int32_t* nflag_out, uint8_t* triggered_out, void* stream) {
  return gg::launch_verify_rows(x_dtype, X, M, K, ldx, y_dtype, Y, N, ldy, chk_prec, w_sum, bias_sum, mu, lo, hi,
                                statistic, d_out, flags_out, max_disc_out, nflag_out, triggered_out,
                                static_cast<cudaStream_t>(stream));
}

size_t gg_b_scratch_bytes(int32_t ab_kind, int64_t N, int64_t K) { return gg::b_scratch_bytes(ab_kind, N, K); }

size_t gg_locate_workspace_bytes(int64_t M, int64_t K) { return gg::locate_workspace_bytes(M, K); }

int gg_locate_tiles(int32_t x_dtype, const void* X, int64_t M, int64_t K, int64_t ldx, const void* W, int64_t N,
                    int64_t ldw, const void* bias, int32_t bias_dtype, int32_t c_dtype, const void* C, int64_t ldc,
                    const uint8_t* flags, const void* d, double mu, double frac, uint8_t* tile_mask, void* col_disc,
                    void* workspace, size_t workspace_bytes, void* stream) {
  return gg::launch_locate_tiles(x_dtype, X, M, K, ldx, W, N, ldw, bias, bias_dtype, c_dtype, C, ldc, flags, d, mu,
                                 frac, tile_mask, col_disc, workspace, workspace_bytes,
                                 static_cast<cudaStream_t>(stream));
}

int gg_flip_bits(void* ptr, int32_t elem_bytes, const int64_t* elem_idx, const int32_t* bit_idx, int64_t n,
                 void* stream) {
  return gg::launch_flip_bits(ptr, elem_bytes, elem_idx, bit_idx, n, static_cast<cudaStream_t>(stream));
}

int gg_gemm_exact(int32_t dtype, int32_t accum, const void* X, int64_t M, int64_t K, const void* Wt, int64_t N,
                  const void* bias, void* Y, void* stream) {
  return gg::launch_gemm_exact(dtype, accum, X, M, K, Wt, N, bias, Y, static_cast<cudaStream_t>(stream));
}

int gg_reduce(int32_t dtype, const void* A, int64_t rows, int64_t cols, int32_t axis, void* out, void* stream) {
  return gg::launch_reduce(dtype, A, rows, cols, axis, out, static_cast<cudaStream_t>(stream));
}

int gg_round_f64_to(int32_t dtype, const double* in, void* out, int64_t n, void* stream) {
  return gg::launch_round(dtype, in, out, n, static_cast<cudaStream_t>(stream));
}

int gg_running_stats(const double* d, int64_t n, double* state, void* stream) {
  return gg::launch_running_stats(d, n, state, static_cast<cudaStream_t>(stream));
}

int gg_minmax(int32_t dtype, const void* Y, int64_t M, int64_t N, int64_t ldy, uint64_t* state, void* stream) {
  return gg::launch_minmax(dtype, Y, M, N, ldy, reinterpret_cast<unsigned long long*>(state),
                           static_cast<cudaStream_t>(stream));
}

int gg_int_finish(const int32_t* Y, int64_t B, int64_t T, int64_t N, int64_t ldy, int32_t relu, int32_t shift,
                  int32_t qkv, int8_t* H, void* stream) {
  return gg::launch_int_finish(Y, B, T, N, ldy, relu, shift, qkv, H, static_cast<cudaStream_t>(stream));
}

int gg_patchify(int32_t dtype, const void* images, int64_t B, int64_t C, int64_t H, int64_t W, int64_t P, void* out,
                void* stream) {
  return gg::launch_patchify(dtype, images, B, C, H, W, P, out, static_cast<cudaStream_t>(stream));
}

int gg_embed_layernorm(int32_t dtype, const void* e, const void* pos, const void* cls, int64_t B, int64_t T,
                       int64_t D, const float* gamma, const float* beta, float eps, void* h_out, void* ln_out,
                       const float* w_pred, uint64_t* pred_out, void* stream) {
  return gg::launch_embed_layernorm(dtype, e, pos, cls, B, T, D, gamma, beta, eps, h_out, ln_out, w_pred,
                                    reinterpret_cast<unsigned long long*>(pred_out), static_cast<cudaStream_t>(stream));
}

int gg_add_layernorm(int32_t dtype, const void* h, const void* y, int64_t rows, int64_t D, const float* gamma,
                     const float* beta, float eps, void* h_out, void* ln_out, const float* w_pred, uint64_t* pred_out,
                     void* stream) {
  return gg::launch_add_layernorm(dtype, h, y, rows, D, gamma, beta, eps, h_out, ln_out, w_pred,
                                  reinterpret_cast<unsigned long long*>(pred_out), static_cast<cudaStream_t>(stream));
}

}  // extern "C"
