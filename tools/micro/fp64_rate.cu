// Throughput of FP64-pipe ops on this GPU: DFMA, DADD, F2F.F64.F32, I2F.F64.S32, FFMA (ref).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(float* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  float f0 = threadIdx.x * 1e-3f, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3, f4 = f0 + 4, f5 = f0 + 5, f6 = f0 + 6, f7 = f0 + 7;
  int i0 = threadIdx.x, i1 = i0 + 1, i2 = i0 + 2, i3 = i0 + 3;
  for (int it = 0; it < iters; ++it) {
    if (OP == 0) { a0 = fma(a0, 1.0000001, 1e-9); a1 = fma(a1, 1.0000001, 1e-9); a2 = fma(a2, 1.0000001, 1e-9); a3 = fma(a3, 1.0000001, 1e-9);
                   a4 = fma(a4, 1.0000001, 1e-9); a5 = fma(a5, 1.0000001, 1e-9); a6 = fma(a6, 1.0000001, 1e-9); a7 = fma(a7, 1.0000001, 1e-9); }
    if (OP == 1) { a0 += (double)f0; a1 += (double)f1; a2 += (double)f2; a3 += (double)f3; a4 += (double)f4; a5 += (double)f5; a6 += (double)f6; a7 += (double)f7;
                   f0 += 1e-7f; f1 += 1e-7f; f2 += 1e-7f; f3 += 1e-7f; f4 += 1e-7f; f5 += 1e-7f; f6 += 1e-7f; f7 += 1e-7f; }
    if (OP == 2) { a0 += (double)i0; a1 += (double)i1; a2 += (double)i2; a3 += (double)i3; i0 += 3; i1 += 3; i2 += 3; i3 += 3; }
    if (OP == 3) { f0 = fmaf(f0, 1.0001f, 1e-7f); f1 = fmaf(f1, 1.0001f, 1e-7f); f2 = fmaf(f2, 1.0001f, 1e-7f); f3 = fmaf(f3, 1.0001f, 1e-7f);
                   f4 = fmaf(f4, 1.0001f, 1e-7f); f5 = fmaf(f5, 1.0001f, 1e-7f); f6 = fmaf(f6, 1.0001f, 1e-7f); f7 = fmaf(f7, 1.0001f, 1e-7f); }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7) + f0 + f1 + f2 + f3 + f4 + f5 + f6 + f7 + i0 + i1 + i2 + i3;
}
template <int OP>
void run(const char* name, int ops_per_iter) {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  int iters = 4096; int blocks = 148 * 4, threads = 512;
  k<OP><<<blocks, threads>>>(out, 16);
  cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
  cudaEventRecord(s); k<OP><<<blocks, threads>>>(out, iters); cudaEventRecord(e); cudaEventSynchronize(e);
  float ms; cudaEventElapsedTime(&ms, s, e);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double ops = double(blocks) * threads * iters * ops_per_iter;
  printf("%-28s %8.3f ms  %10.1f Gop/s  %6.1f op/clk/SM (at %d MHz)\n", name, ms, ops / ms / 1e6, ops / (ms * 1e-3) / (clk * 1e3) / 148, clk / 1000);
  cudaFree(out);
}
int main() {
  run<0>("DFMA", 8);
  run<1>("F2F.F64.F32 + DADD (+FADD)", 8);
  run<2>("I2F.F64.S32 + DADD", 4);
  run<3>("FFMA", 8);
}
