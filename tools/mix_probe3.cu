// Register-tile probe, third series: does more warps per SM (a smaller per-thread tile)
// lift the DPX + IMAD/VIMNMX3 mix above the 8 x 8 tile's 142 (min,+)/clk/SM?
//   R x C accumulators per thread, D of the C columns on DPX, B CTAs of 256 threads per SM.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define OPQ(x) asm volatile("" : "+r"(x))

template <int R, int C, int D, int B>
__global__ void __launch_bounds__(256, B) probe(uint32_t *sink, long long *cyc, int iters, uint32_t one) {
  uint32_t acc[R][C], x0[R], x1[R], b0[C], b1[C];
  uint32_t s = threadIdx.x * 0x00010001u;
#pragma unroll
  for (int i = 0; i < R; ++i) { x0[i] = s + i; x1[i] = s + 2 * i; }
#pragma unroll
  for (int i = 0; i < C; ++i) { b0[i] = s + 3 * i; b1[i] = s + 5 * i; }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[r][c] = 0x3FFF3FFFu;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < R; ++i) { OPQ(x0[i]); OPQ(x1[i]); }
#pragma unroll
    for (int i = 0; i < C; ++i) { OPQ(b0[i]); OPQ(b1[i]); }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (c < D) {
          acc[r][c] = __viaddmin_s16x2(x0[r], b0[c], acc[r][c]);
          acc[r][c] = __viaddmin_s16x2(x1[r], b1[c], acc[r][c]);
        } else {
          const uint32_t p = x0[r] * one + b0[c], q = x1[r] * one + b1[c];
          acc[r][c] = __vimin3_s16x2(acc[r][c], p, q);
        }
      }
  }
  long long t1 = clock64();
  uint32_t h = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) h ^= acc[r][c];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = h;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int R, int C, int D, int B>
void run(int sms) {
  const int blocks = sms * B, threads = 256, iters = 2000;
  uint32_t *sink; long long *cyc;
  cudaMalloc(&sink, blocks * threads * 4);
  cudaMalloc(&cyc, blocks * 8);
  probe<R, C, D, B><<<blocks, threads>>>(sink, cyc, 10, 1);
  probe<R, C, D, B><<<blocks, threads>>>(sink, cyc, iters, 1);
  cudaDeviceSynchronize();
  static long long h[8192];
  cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int b = 0; b < blocks; ++b) mx = h[b] > mx ? h[b] : mx;
  // per SM: B CTAs x 256 threads x R*C accumulators x 4 terms (2 k-pairs) per iteration
  const double per_clk_sm = (double)iters * B * threads * R * C * 4 / (double)mx;
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, probe<R, C, D, B>);
  printf("tile %dx%d DPX cols %d CTAs/SM %d regs %d: %6.1f (min,+)/clk/SM\n", R, C, D, B, a.numRegs, per_clk_sm);
  cudaFree(sink); cudaFree(cyc);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  for (int rep = 0; rep < 2; ++rep) {
    run<8, 8, 3, 2>(sms); run<8, 8, 4, 2>(sms);
    run<8, 4, 2, 3>(sms); run<8, 4, 2, 4>(sms); run<8, 4, 1, 4>(sms); run<8, 4, 2, 2>(sms);
    run<4, 8, 3, 4>(sms); run<4, 8, 4, 4>(sms); run<4, 4, 2, 6>(sms); run<4, 4, 2, 8>(sms);
  }
  return 0;
}
