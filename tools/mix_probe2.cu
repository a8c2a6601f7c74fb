// Register-tile probe, second series: which accumulators take the DPX form and which the
// IMAD(uniform one) + VIMNMX3 form, for the GEMM's 8x8 tile (operands in registers).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mix_probe2 mix_probe2.cu
// PAT 0: columns c < D on DPX | 1: rows r < D on DPX | 2: (r + c) % 8 < D on DPX
// ORD 0: r outer, c inner | 1: c outer, r inner
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define OPQ(x) asm volatile("" : "+r"(x))

template <int PAT, int D, int ORD>
__global__ void __launch_bounds__(256, 2) probe(uint32_t *sink, long long *cyc, int iters, uint32_t one) {
  uint32_t acc[8][8], x0[8], x1[8], b0[8], b1[8];
  uint32_t s = threadIdx.x * 0x00010001u;
#pragma unroll
  for (int i = 0; i < 8; ++i) { x0[i] = s + i; x1[i] = s + 2 * i; b0[i] = s + 3 * i; b1[i] = s + 5 * i; }
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0x3FFF3FFFu;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { OPQ(x0[i]); OPQ(x1[i]); OPQ(b0[i]); OPQ(b1[i]); }
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int r = ORD ? v : u, c = ORD ? u : v;
        const bool dpx = PAT == 0 ? c < D : (PAT == 1 ? r < D : ((r + c) & 7) < D);
        if (dpx) {
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
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) h ^= acc[r][c];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = h;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int PAT, int D, int ORD>
void run(int sms) {
  const int blocks = sms * 2, threads = 256, iters = 2000;
  uint32_t *sink; long long *cyc;
  cudaMalloc(&sink, blocks * threads * 4);
  cudaMalloc(&cyc, blocks * 8);
  probe<PAT, D, ORD><<<blocks, threads>>>(sink, cyc, 10, 1);
  probe<PAT, D, ORD><<<blocks, threads>>>(sink, cyc, iters, 1);
  cudaDeviceSynchronize();
  long long h[4096];
  cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int b = 0; b < blocks; ++b) mx = h[b] > mx ? h[b] : mx;
  const double per_clk_sm = (double)iters * 256 * threads * 2 / (double)mx;
  printf("pattern %s D=%d order %s: %6.1f (min,+)/clk/SM\n", PAT == 0 ? "cols" : (PAT == 1 ? "rows" : "diag"), D,
         ORD ? "c-outer" : "r-outer", per_clk_sm);
  cudaFree(sink); cudaFree(cyc);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  for (int rep = 0; rep < 2; ++rep) {
    run<0, 3, 0>(sms); run<0, 3, 1>(sms); run<0, 4, 0>(sms); run<0, 2, 0>(sms);
    run<1, 3, 0>(sms); run<1, 3, 1>(sms); run<1, 4, 0>(sms); run<1, 2, 0>(sms);
    run<2, 3, 0>(sms); run<2, 4, 0>(sms); run<2, 2, 0>(sms);
  }
  return 0;
}
