// Register-tile probe: the GEMM's 8x8 s16x2 accumulator tile fed from opaque registers
// (no shared memory), for several (min,+) instruction forms.  Reports (min,+) lane-terms
// per SM clock.  Not part of the product; informs the mainloop mix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mix_probe mix_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define OPQ(x) asm volatile("" : "+r"(x))

// FORM: 0 DPX only | 1 IMAD(ur one)+VIMNMX3 | 2 plain '+' + VIMNMX3 | 3 __vadd2 + VIMNMX3
//       4 mix DPXC=3 with IMAD(ur) | 5 mix DPXC=3 with plain '+' | 6 mix DPXC=3 with __vadd2
//       7 mix DPXC=4 plain '+'     | 8 mix DPXC=2 plain '+'
template <int FORM>
__global__ void __launch_bounds__(256, 2) probe(uint32_t *sink, long long *cyc, int iters, uint32_t one) {
  uint32_t acc[8][8], x0[8], x1[8], b0[8], b1[8];
  uint32_t s = threadIdx.x * 0x00010001u;
#pragma unroll
  for (int i = 0; i < 8; ++i) { x0[i] = s + i; x1[i] = s + 2 * i; b0[i] = s + 3 * i; b1[i] = s + 5 * i; }
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0x3FFF3FFFu;
  constexpr int DPXC = FORM == 0 ? 8 : (FORM <= 3 ? 0 : (FORM == 7 ? 4 : (FORM == 8 ? 2 : 3)));
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { OPQ(x0[i]); OPQ(x1[i]); OPQ(b0[i]); OPQ(b1[i]); }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < DPXC) {
          acc[r][c] = __viaddmin_s16x2(x0[r], b0[c], acc[r][c]);
          acc[r][c] = __viaddmin_s16x2(x1[r], b1[c], acc[r][c]);
        } else {
          uint32_t p, q;
          if (FORM == 1 || FORM == 4) { p = x0[r] * one + b0[c]; q = x1[r] * one + b1[c]; }
          else if (FORM == 3 || FORM == 6) { p = __vadd2(x0[r], b0[c]); q = __vadd2(x1[r], b1[c]); }
          else { p = x0[r] + b0[c]; q = x1[r] + b1[c]; }
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

template <int FORM>
void run(int sms, const char *name) {
  const int blocks = sms * 2, threads = 256, iters = 2000;
  uint32_t *sink; long long *cyc;
  cudaMalloc(&sink, blocks * threads * 4);
  cudaMalloc(&cyc, blocks * 8);
  probe<FORM><<<blocks, threads>>>(sink, cyc, 10, 1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<FORM><<<blocks, threads>>>(sink, cyc, iters, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[4096];
  cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int b = 0; b < blocks; ++b) mx = h[b] > mx ? h[b] : mx;
  // per thread per iteration: 64 accumulators x 2 k-pairs x 2 lanes = 256 (min,+) terms
  double per_clk_sm = (double)iters * 256 * threads * 2 / (double)mx;
  printf("form %d %-34s %7.1f (min,+)/clk/SM  = %.3f x DPX-only ceiling (128)   ms=%.2f clk=%.0f MHz\n", FORM,
         name, per_clk_sm, per_clk_sm / 128.0, ms, mx / (ms * 1e3));
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  for (int rep = 0; rep < 2; ++rep) {
    run<0>(sms, "DPX only");
    run<1>(sms, "IMAD(ur one)+VIMNMX3");
    run<2>(sms, "plain + and VIMNMX3");
    run<3>(sms, "__vadd2 + VIMNMX3");
    run<4>(sms, "mix 3/8 DPX, IMAD(ur)");
    run<5>(sms, "mix 3/8 DPX, plain +");
    run<6>(sms, "mix 3/8 DPX, __vadd2");
    run<7>(sms, "mix 4/8 DPX, plain +");
    run<8>(sms, "mix 2/8 DPX, plain +");
  }
  return 0;
}
