// Throughput probe for the integer instructions a (min,+) GEMM can use on sm_100a.
// Measures, per SM per SM-clock, the lane-ops issued by register-only kernels with
// many independent accumulator chains. Used to fix the roofline denominator
// (DESIGN.md "Roofline"); not part of the product path.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o alu_probe alu_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define OPQ(x) asm volatile("" : "+r"(x))

// a*one+b with `one` opaque to the compiler so ptxas keeps IMAD (fma pipe) instead of IADD3
__device__ __forceinline__ uint32_t imad_add(uint32_t a, uint32_t b, uint32_t one) {
  return a * one + b;
}
__device__ __forceinline__ uint32_t iadd(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// MODE: 0 dpx s16x2 | 1 dpx s32 | 2 vimin3 s16x2 | 3 iadd (alu?) | 4 imad add
//       5 (2x imad add + vimin3) | 6 hadd2+hmin2 | 7 dpx + (imad,imad,vimin3) mix 1:1
template <int MODE>
__global__ void __launch_bounds__(256) probe(uint32_t *out, long long *cyc, int iters, uint32_t seed) {
  // 32 accumulators = a 4x8 (i,j) micro-tile; xa*/yb* play the A-column / B-row fragments
  constexpr int U = 32;
  uint32_t c[U], xa0[4], xa1[4], yb0[8], yb1[8];
  uint32_t one = 1u + (seed >> 31);
  uint32_t x0 = (seed ^ threadIdx.x) & 0x000F000Fu;
#pragma unroll
  for (int q = 0; q < 4; ++q) { xa0[q] = x0 + q; xa1[q] = x0 + 2 * q + 1; }
#pragma unroll
  for (int q = 0; q < 8; ++q) { yb0[q] = x0 + 3 * q; yb1[q] = x0 + 5 * q + 2; }
#pragma unroll
  for (int u = 0; u < U; ++u) c[u] = 0x10001000u + u;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    OPQ(one);
#pragma unroll
    for (int q = 0; q < 4; ++q) { OPQ(xa0[q]); OPQ(xa1[q]); }
#pragma unroll
    for (int q = 0; q < 8; ++q) { OPQ(yb0[q]); OPQ(yb1[q]); }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = u >> 3, j = u & 7;
      if (MODE == 0) {         // DPX s16x2, GEMM-shaped operands
        c[u] = __viaddmin_s16x2(xa0[i], yb0[j], c[u]);
      } else if (MODE == 1) {  // DPX s32
        c[u] = (uint32_t)__viaddmin_s32((int)xa0[i], (int)yb0[j], (int)c[u]);
      } else if (MODE == 2) {  // 3-input min only
        c[u] = __vimin3_s16x2(c[u], xa0[i], yb0[j]);
      } else if (MODE == 3) {  // packed add, compiler's choice of opcode
        c[u] = c[u] + xa0[i] + yb0[j];
      } else if (MODE == 4) {  // packed add forced onto IMAD
        c[u] = imad_add(c[u], yb0[j], one);
      } else if (MODE == 5) {  // 2 IMAD adds + VIMNMX3: 2 k-pairs, 4 min-plus lane-ops
        uint32_t s1 = imad_add(xa0[i], yb0[j], one);
        uint32_t s2 = imad_add(xa1[i], yb1[j], one);
        c[u] = __vimin3_s16x2(c[u], s1, s2);
      } else if (MODE == 6) {  // fp16x2 add + min
        __half2 h = __hadd2(*(__half2 *)&xa0[i], *(__half2 *)&yb0[j]);
        __half2 m = __hmin2(h, *(__half2 *)&c[u]);
        c[u] = *(uint32_t *)&m;
      } else if (MODE == 7) {  // 2 plain adds + VIMNMX3 (compiler's add opcode)
        uint32_t s1 = xa0[i] + yb0[j];
        uint32_t s2 = xa1[i] + yb1[j];
        c[u] = __vimin3_s16x2(c[u], s1, s2);
      } else if (MODE == 8) {  // mix: odd u DPX (2 k-pairs as 2 DPX), even u IMAD/IMAD/VIMNMX3
        if (u & 1) {
          c[u] = __viaddmin_s16x2(xa0[i], yb0[j], c[u]);
          c[u] = __viaddmin_s16x2(xa1[i], yb1[j], c[u]);
        } else {
          uint32_t s1 = imad_add(xa0[i], yb0[j], one);
          uint32_t s2 = imad_add(xa1[i], yb1[j], one);
          c[u] = __vimin3_s16x2(c[u], s1, s2);
        }
      }
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) acc ^= c[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// lane-ops of the (min,+) semiring delivered per instruction slot of each mode
// (mode 3/4 deliver an add only; counted as 2 lanes of add for the pipe rate)
static const char *names[] = {"VIADDMNMX.S16x2", "VIADDMNMX s32", "VIMNMX3.S16x2", "add+add (compiler)",
                              "IMAD add", "2xIMAD+VIMNMX3", "HADD2+HMNMX2", "2xadd+VIMNMX3 (compiler)",
                              "mix DPX / IMAD-VIMNMX3"};
// instructions per u per iteration (nominal, from the source)
static const double instr_per_iter_u[] = {1, 1, 1, 2, 1, 3, 2, 3, 2.5};
// (min,+) lane-ops per u per iteration (mode 3/4 do no min: 0)
static const double mp_per_iter_u[] = {2, 1, 0, 0, 0, 4, 2, 4, 4};

template <int MODE>
void run(int sms) {
  int blocks = sms * 4, threads = 256, iters = 4096;
  uint32_t *out; long long *cyc;
  cudaMalloc(&out, blocks * threads * 4);
  cudaMalloc(&cyc, blocks * 8);
  probe<MODE><<<blocks, threads>>>(out, cyc, 16, 1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<MODE><<<blocks, threads>>>(out, cyc, iters, 12345);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long *h = new long long[blocks];
  cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  double avg = 0; long long mx = 0;
  for (int b = 0; b < blocks; ++b) { avg += h[b]; if (h[b] > mx) mx = h[b]; }
  avg /= blocks;
  double warp_instr_per_block = (double)iters * 32 * instr_per_iter_u[MODE] * (threads / 32);
  // 4 blocks per SM co-resident (256 thr, <=64 regs ok): per-SM instr per clock
  double ipc_sm = warp_instr_per_block * 4 / (double)mx;
  double thr_instr = warp_instr_per_block * 32 * blocks;  // thread-instructions
  double mp_per_clk_sm = (double)iters * 32 * mp_per_iter_u[MODE] * threads * 4 / (double)mx;
  double mp_per_s = (double)iters * 32 * mp_per_iter_u[MODE] * threads * blocks / (ms * 1e-3);
  printf("mode %d %-26s ms=%8.3f max_cyc=%9.0f warp-instr/clk/SM=%6.3f minplus/clk/SM=%7.1f minplus/s=%.3e clk_MHz=%.0f\n",
         MODE, names[MODE], ms, (double)mx, ipc_sm, mp_per_clk_sm, mp_per_s, mx / (ms * 1e3));
  (void)avg; (void)thr_instr;
  cudaFree(out); cudaFree(cyc); delete[] h;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs=%d cc=%d.%d clock=%d kHz\n", p.name, p.multiProcessorCount, p.major, p.minor, p.clockRate);
  int sms = p.multiProcessorCount;
  for (int rep = 0; rep < 2; ++rep) {
    run<0>(sms); run<1>(sms); run<2>(sms); run<3>(sms); run<4>(sms); run<5>(sms); run<6>(sms); run<7>(sms); run<8>(sms);
  }
  return 0;
}
