#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#define OPQ(x) asm volatile("" : "+r"(x))
// FORM 0: DPX only; 1: HMNMX2 only; 2: HADD2 only; 3: DPX + HMNMX2 (1:1); 4: DPX + HADD2 (1:1)
// 5: HFMA2 form of add (x*1+b); 6: DPX + (HADD2 + HMNMX2) 2:1 per acc
template <int FORM>
__global__ void __launch_bounds__(256, 2) k(uint32_t *sink, long long *cyc, int iters) {
  uint32_t a[16], b[16], x[4];
  for (int i = 0; i < 16; ++i) { a[i] = threadIdx.x * 3 + i; b[i] = threadIdx.x + 7 * i; }
  for (int i = 0; i < 4; ++i) x[i] = threadIdx.x * 5 + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) OPQ(x[i]);
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (FORM == 0) a[i] = __viaddmin_s16x2(x[u], b[i], a[i]);
      if (FORM == 1) { __half2 h = __hmin2(*(__half2*)&a[i], *(__half2*)&x[u]); a[i] = *(uint32_t*)&h; }
      if (FORM == 2) { __half2 h = __hadd2(*(__half2*)&a[i], *(__half2*)&x[u]); a[i] = *(uint32_t*)&h; }
      if (FORM == 3) {
        if (i & 1) a[i] = __viaddmin_s16x2(x[u], b[i], a[i]);
        else { __half2 h = __hmin2(*(__half2*)&a[i], *(__half2*)&b[i]); a[i] = *(uint32_t*)&h; }
      }
      if (FORM == 4) {
        if (i & 1) a[i] = __viaddmin_s16x2(x[u], b[i], a[i]);
        else { __half2 h = __hadd2(*(__half2*)&a[i], *(__half2*)&x[u]); a[i] = *(uint32_t*)&h; }
      }
      if (FORM == 5) { __half2 h = __hfma2(*(__half2*)&a[i], *(__half2*)&x[u], *(__half2*)&b[i]); a[i] = *(uint32_t*)&h; }
      if (FORM == 6) {
        if (i % 3 == 0) { __half2 s = __hadd2(*(__half2*)&x[u], *(__half2*)&b[i]);
                          __half2 h = __hmin2(*(__half2*)&a[i], s); a[i] = *(uint32_t*)&h; }
        else a[i] = __viaddmin_s16x2(x[u], b[i], a[i]);
      }
    }
  }
  long long t1 = clock64();
  uint32_t h = 0;
  for (int i = 0; i < 16; ++i) h ^= a[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = h;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int F> void run(int sms, const char *name, double instr_per_iter) {
  int blocks = sms * 2, iters = 4000;
  uint32_t *s; long long *c; cudaMalloc(&s, blocks * 256 * 4); cudaMalloc(&c, blocks * 8);
  k<F><<<blocks, 256>>>(s, c, 10); k<F><<<blocks, 256>>>(s, c, iters); cudaDeviceSynchronize();
  long long h[1024]; cudaMemcpy(h, c, blocks * 8, cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
  double wi = (double)iters * instr_per_iter * 8 * 2 / mx;   // warp-instr / clk / SM (8 warps x 2 CTAs)
  printf("form %d %-28s %.3f warp-instr/clk/SM\n", F, name, wi);
  cudaFree(s); cudaFree(c);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int r = 0; r < 2; ++r) {
    run<0>(sms, "DPX", 64); run<1>(sms, "HMNMX2", 64); run<2>(sms, "HADD2", 64);
    run<3>(sms, "DPX+HMNMX2 1:1", 64); run<4>(sms, "DPX+HADD2 1:1", 64); run<5>(sms, "HFMA2", 64);
    run<6>(sms, "DPX 2 : (HADD2+HMNMX2) 1 per acc", 64 + 64.0 / 3 * 1);
  }
}
