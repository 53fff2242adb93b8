// gg_internal.h — shared host-side plumbing of the C-ABI library.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/gemmguard_b200.h"

namespace gg {

// Records `msg` as the thread's last error and returns `code`.
int fail(int code, const std::string& msg);
// Converts a pending CUDA error (if any) into GG_ECUDA.
int check_launch(const char* what);

inline int dtype_bytes(int dt) {
  switch (dt) {
    case GG_F64: case GG_I64: return 8;
    case GG_F32: case GG_I32: return 4;
    case GG_F16: case GG_BF16: return 2;
    case GG_I8: return 1;
    default: return 0;
  }
}
inline int prec_bytes(int p) {
  switch (p) {
    case GG_P_F16: return 2;
    case GG_P_F32: return 4;
    case GG_P_F64: case GG_P_I64: return 8;
    default: return 0;
  }
}

// launchers implemented in gg_aux.cu
int launch_offline_checksum(int w_dtype, const void* W, int64_t K, int64_t N, int64_t ldw, int w_layout,
                            const void* bias, int bias_dtype, int chk_prec, void* w_sum_out, void* bias_sum_out,
                            cudaStream_t s);
int launch_verify_rows(int x_dtype, const void* X, int64_t M, int64_t K, int64_t ldx, int y_dtype, const void* Y,
                       int64_t N, int64_t ldy, int chk_prec, const void* w_sum, const void* bias_sum, double mu,
                       double lo, double hi, int statistic, void* d_out, uint8_t* flags_out, double* max_disc_out,
                       int32_t* nflag_out, uint8_t* triggered_out, cudaStream_t s);
int launch_flip_bits(void* ptr, int elem_bytes, const int64_t* elem_idx, const int32_t* bit_idx, int64_t n,
                     cudaStream_t s);
int launch_gemm_exact(int dtype, int accum, const void* X, int64_t M, int64_t K, const void* Wt, int64_t N,
                      const void* bias, void* Y, cudaStream_t s);
int launch_reduce(int dtype, const void* A, int64_t rows, int64_t cols, int axis, void* out, cudaStream_t s);
// batch_mean statistic of a protected launch: flags / summaries from every d (pairwise mean)
int launch_batch_mean_finish(int64_t M, double mu, double lo, double hi, const double* d, uint8_t* flags,
                             double* max_disc, int32_t* nflag, uint8_t* triggered, cudaStream_t s);
int launch_round(int dtype, const double* in, void* out, int64_t n, cudaStream_t s);

size_t checksum_aux_bytes(int ab_kind, int64_t K);
int launch_split_tf32x3(const float* src, int64_t rows, int64_t K, int64_t ld, int role, float* dst, int64_t ldd,
                        cudaStream_t s);
int launch_checksum_aux(int ab_kind, const void* w_sum, int64_t K, void* aux, cudaStream_t s);

// implemented in gg_calib.cu
int launch_running_stats(const double* d, int64_t n, double* state, cudaStream_t s);
int launch_minmax(int dtype, const void* Y, int64_t M, int64_t N, int64_t ldy, unsigned long long* state,
                  cudaStream_t s);

// implemented in gg_toy.cu
int launch_int_finish(const int* y, int64_t B, int64_t T, int64_t N, int64_t ldy, int relu, int shift, int qkv,
                      int8_t* h, cudaStream_t s);

// implemented in gg_vit.cu
int launch_add_layernorm(int dtype, const void* h, const void* y, int64_t rows, int64_t D, const float* gamma,
                         const float* beta, float eps, void* h_out, void* ln_out, const float* w_pred,
                         unsigned long long* pred_out, cudaStream_t s);

int launch_patchify(int dtype, const void* images, int64_t B, int64_t C, int64_t H, int64_t W, int64_t P, void* out,
                    cudaStream_t s);
int launch_embed_layernorm(int dtype, const void* e, const void* pos, const void* cls, int64_t B, int64_t T,
                           int64_t D, const float* gamma, const float* beta, float eps, void* h_out, void* ln_out,
                           const float* w_pred, unsigned long long* pred_out, cudaStream_t s);

// implemented in gg_locate.cu
size_t locate_workspace_bytes(int64_t M, int64_t K);
int launch_locate_tiles(int x_dtype, const void* X, int64_t M, int64_t K, int64_t ldx, const void* W, int64_t N,
                        int64_t ldw, const void* bias, int bias_dtype, int c_dtype, const void* C, int64_t ldc,
                        const uint8_t* flags, const void* d, double mu, double frac, uint8_t* tile_mask,
                        void* col_disc, void* workspace, size_t workspace_bytes, cudaStream_t s);

// implemented in gg_gemm_sm100.cu
size_t protected_gemm_workspace_bytes(int64_t M, int64_t N);
size_t b_scratch_bytes(int ab_kind, int64_t N, int64_t K);
int launch_protected_gemm(const gg_gemm_desc* d, bool replay, cudaStream_t s);

}  // namespace gg
