// Register-tile probe of a third add form for the (min,+) mainloop (not part of the product;
// informs the mix).  HADD2 on raw int16 bit patterns is the exact integer sum
// while operands and sum stay below 2048: a value k < 2048 read as fp16 is k * 2^-24 (the
// subnormals and the first binade), whose bit pattern is k; RD_INF = 0x3FFF plus any such k
// rounds back to 0x3FFF.  So s = HADD2(x, b) can stand in for the IMAD packed add on the same
// operands.  The question is whether HADD2 issues beside IMAD (the other fma sub-pipe).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hadd_probe hadd_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define OPQ(x) asm volatile("" : "+r"(x))

__device__ __forceinline__ uint32_t hadd2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("add.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// FORM 0: independent IMAD chains (packed int add via x*one+b)   -> instr/clk
// FORM 1: independent HADD2 chains                                  -> instr/clk
// FORM 2: independent FFMA chains                                   -> instr/clk
// FORM 3: GEMM 8x8 tile, every column [2 HADD2 + VIMNMX3.U16x2]     -> terms/clk
// FORM 4: GEMM 8x8 tile, d=3 DPX + 5 x [2 IMAD + VIMNMX3] (today's mix)
// FORM 5: GEMM 8x8 tile, 4 x [2 IMAD + VIMNMX3] + 4 x [2 HADD2 + VIMNMX3]
// FORM 6: GEMM 8x8 tile, 3 DPX + 2 x [2 IMAD + VIMNMX3] + 3 x [2 HADD2 + VIMNMX3]
// FORM 7: GEMM 8x8 tile, 3 DPX + 5 x [2 HADD2 + VIMNMX3]
// FORM 8: GEMM 8x8 tile, 2 DPX + 3 x [IMAD] + 3 x [HADD2]
// FORM 9: GEMM 8x8 tile, 4 DPX + 2 x [IMAD] + 2 x [HADD2]
// (HADD2 on int16 bit patterns is the exact integer sum below 2048: a value k < 2048 read as
// fp16 is the subnormal/first-binade number k * 2^-24 whose bit pattern is k.)
template <int FORM>
__global__ void __launch_bounds__(256, 2) probe(uint32_t *sink, long long *cyc, int iters, uint32_t one) {
  long long t0 = 0, t1 = 0;
  uint32_t h = 0;
  if (FORM <= 2) {
    uint32_t c[32], a0[4], b0[8];
    const uint32_t s = (one ^ threadIdx.x) & 0x000F000Fu;
#pragma unroll
    for (int q = 0; q < 4; ++q) a0[q] = 0x3C003C00u + s + q;
#pragma unroll
    for (int q = 0; q < 8; ++q) b0[q] = 0x3C003C00u + s + 3 * q;
#pragma unroll
    for (int u = 0; u < 32; ++u) c[u] = 0x10001000u + u;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int q = 0; q < 4; ++q) OPQ(a0[q]);
#pragma unroll
      for (int q = 0; q < 8; ++q) OPQ(b0[q]);
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        if (FORM == 0) c[u] = a0[u >> 3] * one + c[u];
        else if (FORM == 1) c[u] = hadd2(b0[u & 7], c[u]);
        else c[u] = __float_as_uint(fmaf(__uint_as_float(a0[u >> 3]), __uint_as_float(b0[u & 7]), __uint_as_float(c[u])));
      }
    }
    t1 = clock64();
#pragma unroll
    for (int u = 0; u < 32; ++u) h ^= c[u];
  } else {
    uint32_t acc[8][8], x0[8], x1[8], b0[8], b1[8];
    const uint32_t s = threadIdx.x * 0x00010001u;
#pragma unroll
    for (int i = 0; i < 8; ++i) { x0[i] = s + i; x1[i] = s + 2 * i; b0[i] = s + 3 * i; b1[i] = s + 5 * i; }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = 0x3FFF3FFFu;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) { OPQ(x0[i]); OPQ(x1[i]); OPQ(b0[i]); OPQ(b1[i]); }
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          constexpr int D = FORM == 4 || FORM == 6 || FORM == 7 ? 3 : (FORM == 8 ? 2 : (FORM == 9 ? 4 : 0));
          const bool h16 = FORM == 3 || (FORM == 5 && c >= 4) || (FORM == 6 && c >= 5) || (FORM == 7 && c >= 3) ||
                           (FORM == 8 && c >= 5) || (FORM == 9 && c >= 6);
          if (c < D) {
            acc[r][c] = __viaddmin_s16x2(x0[r], b0[c], acc[r][c]);
            acc[r][c] = __viaddmin_s16x2(x1[r], b1[c], acc[r][c]);
          } else if (h16) {
            acc[r][c] = __vimin3_u16x2(acc[r][c], hadd2(x0[r], b0[c]), hadd2(x1[r], b1[c]));
          } else {
            acc[r][c] = __vimin3_s16x2(acc[r][c], x0[r] * one + b0[c], x1[r] * one + b1[c]);
          }
        }
    }
    t1 = clock64();
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) h ^= acc[r][c];
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = h;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// FORM 10: three k-pairs per step, every column [3 IMAD + VIMNMX3(s0,s1,s2) + VIMNMX(acc, m)]
// FORM 11: three k-pairs per step, 3 DPX columns (3 DPX each) + 5 columns as FORM 10
template <int FORM>
__global__ void __launch_bounds__(256, 2) probe3(uint32_t *sink, long long *cyc, int iters, uint32_t one) {
  uint32_t acc[8][8], x0[8], x1[8], x2[8], b0[8], b1[8], b2[8];
  const uint32_t s = threadIdx.x * 0x00010001u;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x0[i] = s + i; x1[i] = s + 2 * i; x2[i] = s + 7 * i; b0[i] = s + 3 * i; b1[i] = s + 5 * i; b2[i] = s + 11 * i;
  }
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0x3FFF3FFFu;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { OPQ(x0[i]); OPQ(x1[i]); OPQ(x2[i]); OPQ(b0[i]); OPQ(b1[i]); OPQ(b2[i]); }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (FORM == 11 && c < 3) {
          acc[r][c] = __viaddmin_s16x2(x0[r], b0[c], acc[r][c]);
          acc[r][c] = __viaddmin_s16x2(x1[r], b1[c], acc[r][c]);
          acc[r][c] = __viaddmin_s16x2(x2[r], b2[c], acc[r][c]);
        } else {
          const uint32_t m = __vimin3_s16x2(x0[r] * one + b0[c], x1[r] * one + b1[c], x2[r] * one + b2[c]);
          acc[r][c] = __vmins2(acc[r][c], m);
        }
      }
  }
  const long long t1 = clock64();
  uint32_t h = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) h ^= acc[r][c];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = h;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int FORM>
void run3(int sms, const char *name) {
  const int blocks = sms * 2, threads = 256, iters = 2000;
  uint32_t *sink;
  long long *cyc;
  cudaMalloc(&sink, blocks * threads * 4);
  cudaMalloc(&cyc, blocks * 8);
  probe3<FORM><<<blocks, threads>>>(sink, cyc, 16, 1);
  probe3<FORM><<<blocks, threads>>>(sink, cyc, iters, 1);
  cudaDeviceSynchronize();
  long long *h = new long long[blocks];
  cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int b = 0; b < blocks; ++b) mx = h[b] > mx ? h[b] : mx;
  const double t = (double)iters * 384.0 * threads * 2 / (double)mx;   // 64 acc x 3 k-pairs x 2 lanes
  printf("%-44s %.1f (min,+) terms/clk/SM\n", name, t);
  delete[] h;
  cudaFree(sink);
  cudaFree(cyc);
}

template <int FORM>
void run(int sms, const char *name) {
  const int blocks = sms * 2, threads = 256, iters = FORM <= 2 ? 8192 : 2000;
  uint32_t *sink;
  long long *cyc;
  cudaMalloc(&sink, blocks * threads * 4);
  cudaMalloc(&cyc, blocks * 8);
  probe<FORM><<<blocks, threads>>>(sink, cyc, 16, 1);
  probe<FORM><<<blocks, threads>>>(sink, cyc, iters, 1);
  cudaDeviceSynchronize();
  long long *h = new long long[blocks];
  cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int b = 0; b < blocks; ++b) mx = h[b] > mx ? h[b] : mx;
  if (FORM <= 2) {
    const double ipc = (double)iters * 32 * (threads / 32) * 2 / (double)mx;
    printf("%-44s %.3f warp-instr/clk/SM\n", name, ipc);
  } else {
    const double t = (double)iters * 256.0 * threads * 2 / (double)mx;
    printf("%-44s %.1f (min,+) terms/clk/SM\n", name, t);
  }
  delete[] h;
  cudaFree(sink);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>(sms, "IMAD packed add (independent)");
  run<1>(sms, "HADD2 (independent)");
  run<2>(sms, "FFMA (independent)");
  run<3>(sms, "8x8 tile: all [2 HADD2 + VIMNMX3.U16x2]");
  run<4>(sms, "8x8 tile: 3 DPX + 5 [2 IMAD + VIMNMX3] (GEMM)");
  run<5>(sms, "8x8 tile: 4 [IMAD] + 4 [HADD2] groups");
  run<6>(sms, "8x8 tile: 3 DPX + 2 [IMAD] + 3 [HADD2]");
  run<7>(sms, "8x8 tile: 3 DPX + 5 [HADD2]");
  run<8>(sms, "8x8 tile: 2 DPX + 3 [IMAD] + 3 [HADD2]");
  run<9>(sms, "8x8 tile: 4 DPX + 2 [IMAD] + 2 [HADD2]");
  run3<10>(sms, "8x8 tile, 3 k-pairs: all [3 IMAD + V3 + VMIN]");
  run3<11>(sms, "8x8 tile, 3 k-pairs: 3 DPX + 5 [3 IMAD+V3+VMIN]");
  return 0;
}
