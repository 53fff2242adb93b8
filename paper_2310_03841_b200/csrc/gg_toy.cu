// gg_toy.cu — device glue of the integer toy pipeline.
//
// model.finish_layer_output for integer models (model.py:307-331) turns a layer's raw
// int32 GEMM output into the next int8 hidden state:
//   relu (mlp_fc1)                    h = max(y, 0)
//   requantise                        h = clip((h + 2^(s-1)) >> s, -128, 127),
//                                     s = 2 + floor(log2(in_dim)) / 2      (model.py:312-316)
//   qkv: head mixing                  m = floor((q + k + v) / 3)
//        token mixing                 h = floor((m + floor(sum_t m / T)) / 2)  (model.py:298-304)
// gg_int_finish does this for B samples of T tokens at once, so a batched forward keeps
// the hidden state on the device between protected GEMMs.  Integer arithmetic with
// NumPy's semantics (int32 wrap-around, arithmetic shift, floor division): bit-exact.
#include <cuda_runtime.h>

#include <cstdint>

#include "gg_internal.h"

namespace gg {
namespace {

__device__ __forceinline__ long long floor_div(long long a, long long b) {  // b > 0
  long long q = a / b;
  if ((a % b) != 0 && a < 0) --q;
  return q;
}

__device__ __forceinline__ int requant(int y, bool relu, int shift) {
  int h = relu ? max(y, 0) : y;
  h = static_cast<int>(static_cast<unsigned>(h) + (1u << (shift - 1)));  // int32 wrap, like NumPy
  h >>= shift;                                                            // arithmetic shift
  return min(max(h, -128), 127);
}

// Elementwise layers: h[r, c] = requant(y[r, c]).
__global__ void int_finish_kernel(const int* y, int64_t rows, int64_t N, int64_t ldy, bool relu, int shift,
                                  int8_t* h) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < rows * N; e += stride) {
    const int64_t r = e / N, c = e - r * N;
    h[e] = static_cast<int8_t>(requant(y[r * ldy + c], relu, shift));
  }
}

// qkv layers: one thread per (sample, column c < N/3) walks the sample's T tokens twice.
__global__ void int_qkv_mix_kernel(const int* y, int64_t B, int64_t T, int64_t N, int64_t ldy, int shift,
                                   int8_t* h) {
  const int64_t d = N / 3;
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t b = blockIdx.y;
  if (c >= d || b >= B) return;
  const int* yb = y + b * T * ldy;
  auto head_mix = [&](int64_t t) -> long long {  // floor((q + k + v) / 3) of the requantised q, k, v
    const int* row = yb + t * ldy;
    const long long s3 = static_cast<long long>(requant(row[c], false, shift)) + requant(row[c + d], false, shift) +
                         requant(row[c + 2 * d], false, shift);
    return floor_div(s3, 3);
  };
  long long col = 0;
  for (int64_t t = 0; t < T; ++t) col += head_mix(t);
  const long long mean = floor_div(col, T);
  int8_t* hb = h + b * T * d;
  for (int64_t t = 0; t < T; ++t) hb[t * d + c] = static_cast<int8_t>(floor_div(head_mix(t) + mean, 2));
}

}  // namespace

int launch_int_finish(const int* y, int64_t B, int64_t T, int64_t N, int64_t ldy, int relu, int shift, int qkv,
                      int8_t* h, cudaStream_t s) {
  if (B < 1 || T < 1 || N < 1 || ldy < N) return fail(GG_EINVAL, "int_finish: bad shape");
  if (y == nullptr || h == nullptr) return fail(GG_EINVAL, "int_finish: null pointer");
  if (shift < 1 || shift > 30) return fail(GG_EINVAL, "int_finish: requant shift out of range");
  if (qkv) {
    if (N % 3) return fail(GG_EINVAL, "int_finish: qkv width must be divisible by 3");
    const int64_t d = N / 3;
    dim3 grid(static_cast<unsigned>((d + 127) / 128), static_cast<unsigned>(B));
    int_qkv_mix_kernel<<<grid, 128, 0, s>>>(y, B, T, N, ldy, shift, h);
  } else {
    const int64_t n = B * T * N;
    const int64_t blocks = (n + 255) / 256;
    int_finish_kernel<<<static_cast<unsigned>(blocks < 4096 ? blocks : 4096), 256, 0, s>>>(y, B * T, N, ldy,
                                                                                            relu != 0, shift, h);
  }
  return check_launch("int_finish");
}

}  // namespace gg
