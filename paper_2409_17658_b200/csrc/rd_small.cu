// Device-resident Algorithm 2 for small orders (N <= kSmallMaxN: m <= 6), DESIGN.md §5
// "Small orders".
//
// At m = 3..6 a power step is 3.6e4 .. 6.1e8 (min,+) terms — microseconds of GPU work — so a
// host-driven chain (a launch, a stats D2H and a host decision per power) is bound by launch
// and synchronisation latency.  Here ONE cooperative kernel runs the whole of Algorithm 2
// (P:282-298): it packs A, computes A^k = A^{k-1} (x) A (Alg 2 step 3) tile by tile with
// DPX VIADDMNMX.S16x2 on k-pairs, fuses the diagonal min (Cor 7) and the
// periodicity test A^k = beta (x) A^{k-alpha} (Alg 2 step 4; Prop 8) into the tile
// epilogue, meets at a grid barrier, and every CTA takes the same decision from the reduced
// stats (first detection, smallest alpha; or the paper-compatible policy, R6).
// The host reads one result block at the end.
//
// Layout (private to this path): powers are row-major int16 with pitch P (N rounded up to
// 64), +inf = RD_INF, padding INF, in a ring of alpha_max + 1 slots (<= 17.6 MB at m = 6:
// L2-resident).  The right operand A is packed in k-pairs BP[t][j] = A[2t][j] | A[2t+1][j] << 16
// so that the left operand's (X[i][2t], X[i][2t+1]) is one 32-bit word of its row.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>

#include "rd_gemm.cuh"
#include "rd_internal.h"

namespace rd {
namespace {

constexpr int kST = 64;          // output tile (rows and columns)
constexpr int kSThreads = 256;   // 16 x 16 threads, 4 x 4 outputs each
constexpr int kSKC = 32;         // k-pairs per shared-memory chunk

struct SmallArgs {
  const int16_t *A;   // N x N row-major, entries in [0, RD_INF]
  int64_t N, P;       // order, pitch (multiple of kST)
  uint32_t *BP;       // [P/2][P] packed right operand
  int16_t *ring;      // (alpha_max + 1) slots of P x P
  int32_t *stats;     // (kmax + 1) x (1 + 4 alpha_max) MIN-reducible stats, per power
  int32_t *result;    // [found, n0, alpha, beta, k_stop, diag1, diag[0..kmax]]
  unsigned *bar;      // grid barrier: [count, generation]
  int kmax, alpha_max, policy;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Sense-free grid barrier over a cooperative launch (all CTAs co-resident): the last CTA to
// arrive resets the count and bumps the generation; the others spin on the generation.
__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned &gen) {
  __syncthreads();
  if (gridDim.x == 1) return;   // one CTA (m <= 3): the block barrier orders its global writes
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned g = gen;
    if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(&bar[1], 1u);
    } else {
      while (ld_acquire(&bar[1]) == g) {
      }
    }
    __threadfence();
  }
  ++gen;
  __syncthreads();
}

// Loads of data written earlier in the same launch: ld.global.cg (L2, coherent across CTAs);
// a one-CTA grid reads through L1 (its own writes, ordered by the block barrier).
template <bool ONE, typename T>
__device__ __forceinline__ T ldc(const T *p) {
  if constexpr (ONE) return *p;
  else return __ldcg(p);
}

// Alg 2 step 4 on a reduced stats vector (same rule as rd_stats_decide, rd_host.cpp).
template <bool ONE>
__device__ __forceinline__ bool decide(const int32_t *s, int alpha_max, int k, int only, int &alpha, int &beta) {
  const int amax = min(alpha_max, k - 1);
  for (int a = 1; a <= amax; ++a) {
    if (only > 0 && a != only) continue;
    const int32_t *e = s + 1 + 4 * (a - 1);
    const int32_t lo = ldc<ONE>(e), mhi = ldc<ONE>(e + 1), mis = ldc<ONE>(e + 2), fin = ldc<ONE>(e + 3);
    if (mis == 0 && fin != 0 && (int64_t)lo == -(int64_t)mhi && lo >= 0) {
      alpha = a;
      beta = lo;
      return true;
    }
  }
  return false;
}

template <bool ONE>
__global__ void __launch_bounds__(kSThreads, 2) small_chain_kernel(SmallArgs sa) {
  __shared__ __align__(16) uint32_t sX[2][kST][kSKC];   // [row][k-pair]
  __shared__ __align__(16) uint32_t sB[2][kSKC][kST];   // [k-pair][column]
  __shared__ int32_t red[kSThreads / 32][1 + 4 * kMaxAlpha];
  __shared__ int s_stop;
  __shared__ int32_t s_st[1 + 4 * kMaxAlpha];   // one-CTA grid: the power's stats in shared memory
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t N = sa.N, P = sa.P, P2 = P / 2;
  const int am = sa.alpha_max, slen = 1 + 4 * am;
  const int64_t slot_elems = P * P;
  unsigned gen = 0;
  auto slot = [&](int k) { return sa.ring + (int64_t)(k % (am + 1)) * slot_elems; };

  // ---- prologue: pack A, A^1 into its slot, INF elsewhere, neutral stats for every power
  // (sizes fit 32-bit indices: P <= 1024, (alpha_max + 1) P^2 <= 34.6e6)
  {
    const int nth = gridDim.x * blockDim.x, t0 = blockIdx.x * blockDim.x + tid;
    const int n = (int)N, p = (int)P, p2 = (int)P2, se = (int)slot_elems;
    for (int e = t0; e < p2 * p; e += nth) {
      const int t = e / p, j = e - t * p;
      uint32_t lo = RD_INF, hi = RD_INF;
      if (j < n) {
        if (2 * t < n) lo = (uint32_t)min((int)sa.A[2 * t * n + j], (int)RD_INF);
        if (2 * t + 1 < n) hi = (uint32_t)min((int)sa.A[(2 * t + 1) * n + j], (int)RD_INF);
      }
      sa.BP[e] = lo | (hi << 16);
    }
    const int s1 = 1 % (am + 1);
    uint32_t *ring32 = reinterpret_cast<uint32_t *>(sa.ring);
    for (int e = t0; e < (am + 1) * se / 2; e += nth) {
      const int s = (2 * e) / se, r = 2 * e - s * se, i = r / p, j = r - i * p;   // j even
      uint32_t v = kInf2;
      if (s == s1 && i < n) {
        const uint32_t lo = j < n ? (uint32_t)min((int)sa.A[i * n + j], (int)RD_INF) : RD_INF;
        const uint32_t hi = j + 1 < n ? (uint32_t)min((int)sa.A[i * n + j + 1], (int)RD_INF) : RD_INF;
        v = lo | (hi << 16);
      }
      ring32[e] = v;
    }
    for (int e = t0; e < (sa.kmax + 1) * slen; e += nth) {
      const int q = e % slen;
      sa.stats[e] = (q == 0 || (q - 1) % 4 < 2) ? INT_MAX : 0;
    }
    if (blockIdx.x == 0 && warp == 0) {
      if (tid == 0) { sa.result[0] = 0; sa.result[1] = 0; sa.result[2] = 0; sa.result[3] = 0; sa.result[4] = 0; }
      int32_t d1 = INT_MAX;
      for (int q = lane; q < n; q += 32) {
        const int v = sa.A[q * n + q];
        if (v < RD_INF) d1 = min(d1, v);
      }
      d1 = __reduce_min_sync(0xffffffffu, d1);
      if (lane == 0) sa.result[5] = d1;
    }
  }
  grid_barrier(sa.bar, gen);

  const int ty = tid >> 4, tx = tid & 15;   // rows ty*4 + 0..3, columns tx*4 + 0..3
  const int ntile = (int)(P / kST), ntiles = ntile * ntile;
  const int nchunk = (int)((P2 + kSKC - 1) / kSKC);
  int found_k = -1, n0 = 0, al = 0, be = 0, k_stop = sa.kmax;
  for (int k = 2; k <= sa.kmax; ++k) {
    const int16_t *X = slot(k - 1);
    int16_t *C = slot(k);
    const int nprev = min(am, k - 1);
    int32_t *st = sa.stats + (int64_t)k * slen;
    if constexpr (ONE) {   // a lone CTA reduces and decides in shared memory (no global atomics)
      st = s_st;
      for (int e = tid; e < slen; e += kSThreads) s_st[e] = (e == 0 || (e - 1) % 4 < 2) ? INT_MAX : 0;
      __syncthreads();
    }
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t i0 = (int64_t)(tile / ntile) * kST, j0 = (int64_t)(tile % ntile) * kST;
      uint32_t acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = kInf2;
      // chunk = 64 rows x 32 k-pairs of X (row-major words) and 32 k-pairs x 64 columns of BP:
      // 8 + 8 words per thread, fetched into registers one chunk ahead of the compute
      constexpr int kQ = (kSKC * kST) / kSThreads;
      uint32_t px[kQ], pb[kQ];
      auto fetch = [&](int ch) {
        const int64_t t0 = (int64_t)ch * kSKC;
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
          const int e = q * kSThreads + tid;
          const int r = e / kSKC, tp = e % kSKC;   // consecutive threads: consecutive k-pairs of a row
          px[q] = t0 + tp < P2 ? ldc<ONE>(reinterpret_cast<const uint32_t *>(X + (i0 + r) * P) + t0 + tp) : kInf2;
          const int bt = e / kST, bc = e % kST;    // consecutive threads: consecutive columns
          pb[q] = t0 + bt < P2 ? ldc<ONE>(sa.BP + (t0 + bt) * P + j0 + bc) : kInf2;
        }
      };
      auto stash = [&](int buf) {
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
          const int e = q * kSThreads + tid;
          sX[buf][e / kSKC][e % kSKC] = px[q];
          sB[buf][e / kST][e % kST] = pb[q];
        }
      };
      fetch(0);
      stash(0);
      __syncthreads();
      for (int ch = 0; ch < nchunk; ++ch) {
        const int buf = ch & 1;
        if (ch + 1 < nchunk) fetch(ch + 1);
#pragma unroll 2
        for (int t4 = 0; t4 < kSKC / 4; ++t4) {
          uint4 xr[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) xr[r] = *reinterpret_cast<const uint4 *>(&sX[buf][ty * 4 + r][t4 * 4]);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint4 ba = *reinterpret_cast<const uint4 *>(&sB[buf][t4 * 4 + q][tx * 4]);
            const uint32_t b[4] = {ba.x, ba.y, ba.z, ba.w};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const uint32_t x = q == 0 ? xr[r].x : q == 1 ? xr[r].y : q == 2 ? xr[r].z : xr[r].w;
#pragma unroll
              for (int c = 0; c < 4; ++c) acc[r][c] = __viaddmin_s16x2(x, b[c], acc[r][c]);
            }
          }
        }
        if (ch + 1 < nchunk) stash(buf ^ 1);
        __syncthreads();
      }
      // epilogue: fold the k-pair lanes, store row-major int16, diag and stats vs the ring
      uint32_t out[4][2];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const uint32_t a0 = acc[r][2 * p], a1 = acc[r][2 * p + 1];
          out[r][p] = __vmins2(prmt(a0, a1, 0x5410), prmt(a0, a1, 0x7632));
        }
      // the tile goes to its ring slot and, as words, to shared memory (the chunk buffers are
      // free after the k loop's last barrier) for the periodicity stats below
      uint32_t(*sC)[kST / 2] = reinterpret_cast<uint32_t(*)[kST / 2]>(&sX[0][0][0]);
      int32_t dmin = INT_MAX;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int64_t i = i0 + ty * 4 + r, j = j0 + tx * 4;
        *reinterpret_cast<uint2 *>(C + i * P + j) = make_uint2(out[r][0], out[r][1]);
        *reinterpret_cast<uint2 *>(&sC[ty * 4 + r][tx * 2]) = make_uint2(out[r][0], out[r][1]);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (i == j + c) dmin = min(dmin, (int)((out[r][c >> 1] >> (16 * (c & 1))) & 0xFFFF));
      }
      dmin = __reduce_min_sync(0xffffffffu, dmin);
      if (lane == 0) red[warp][0] = dmin;
      __syncthreads();
      // periodicity stats: warp w takes alpha = 1 + w, 1 + w + 8, ...; a lane compares 16
      // 16-byte chunks of the tile (from shared memory) with the same chunks of A^{k-alpha},
      // all 16 loads in flight at once
      for (int a = 1 + warp; a <= nprev; a += kSThreads / 32) {
        const int16_t *Pv = slot(k - a);
        uint32_t lo2 = 0x7FFF7FFFu, hi2 = 0x80008000u, mis = 0, fin = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint4 pv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int q = lane + 32 * (8 * h + u), row = q >> 3, c8 = q & 7;
            pv[u] = ldc<ONE>(reinterpret_cast<const uint4 *>(Pv + (i0 + row) * P + j0 + c8 * 8));
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int q = lane + 32 * (8 * h + u), row = q >> 3, c8 = q & 7;
            const uint4 cv = *reinterpret_cast<const uint4 *>(&sC[row][c8 * 4]);
            stats_pair(cv.x, pv[u].x, lo2, hi2, mis, fin);
            stats_pair(cv.y, pv[u].y, lo2, hi2, mis, fin);
            stats_pair(cv.z, pv[u].z, lo2, hi2, mis, fin);
            stats_pair(cv.w, pv[u].w, lo2, hi2, mis, fin);
          }
        }
        int32_t lo = min((int32_t)(int16_t)(lo2 & 0xFFFF), (int32_t)(int16_t)(lo2 >> 16));
        int32_t hi = max((int32_t)(int16_t)(hi2 & 0xFFFF), (int32_t)(int16_t)(hi2 >> 16));
        if (!(fin & 0xFFFF) && !(fin >> 16)) { lo = INT_MAX; hi = INT_MIN + 1; }
        const int32_t v0 = __reduce_min_sync(0xffffffffu, lo), v1 = __reduce_min_sync(0xffffffffu, -hi);
        const int32_t v2 = __reduce_min_sync(0xffffffffu, mis ? -1 : 0);
        const int32_t v3 = __reduce_min_sync(0xffffffffu, fin ? -1 : 0);
        if (lane == 0) {
          atomicMin(st + 4 * a - 3, v0); atomicMin(st + 4 * a - 2, v1);
          atomicMin(st + 4 * a - 1, v2); atomicMin(st + 4 * a, v3);
        }
      }
      if (tid == 0) {
        int32_t v = red[0][0];
#pragma unroll
        for (int w = 1; w < kSThreads / 32; ++w) v = min(v, red[w][0]);
        atomicMin(st, v);
      }
      __syncthreads();
    }
    grid_barrier(sa.bar, gen);
    // Algorithm 2's decision, taken identically by every CTA on the reduced stats of A^k
    if (tid == 0) {
      int a = 0, b = 0;
      int stop = 0;
      if (found_k < 0) {
        if (decide<ONE>(st, am, k, 0, a, b)) {
          found_k = k; n0 = k - a; al = a; be = b;
          if (sa.policy == 0) stop = 1;
        }
      } else {
        const int aa = k - n0;
        if (aa <= am && decide<ONE>(st, am, k, aa, a, b)) { al = a; be = b; }
        if (aa >= am) stop = 1;
      }
      s_stop = stop;
      if (blockIdx.x == 0) {
        const int32_t d = ldc<ONE>(st);
        sa.result[6 + k] = d >= RD_INF ? INT_MAX : d;
      }
    }
    __syncthreads();
    if (s_stop) { k_stop = k; break; }
  }
  if (blockIdx.x == 0 && tid == 0) {
    sa.result[0] = found_k >= 0;
    sa.result[1] = n0; sa.result[2] = al; sa.result[3] = be; sa.result[4] = k_stop;
  }
}

}  // namespace

// Runs Algorithm 2 for the host matrix A (N x N int16, entries in [0, RD_INF]) as one
// device-resident kernel; t_chain = launch to result on the host.
int small_power_sequence(const int16_t *Ahost, int64_t N, int kmax, int alpha_max, int policy, rd_period_t *out,
                         int32_t *diag, double *t_build, double *t_chain) {
  if (N < 1 || N > kSmallMaxN) return fail(RD_EINVAL, "small_power_sequence: N=%lld out of 1..%d", (long long)N, kSmallMaxN);
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t P = round_up(N, kST);
  const int slen = 1 + 4 * alpha_max;
  // one non-blocking stream per host thread and device, kept for the process: creating and
  // destroying a stream per call cost more than the whole chain at m = 3
  static thread_local cudaStream_t s_st[64] = {};
  int sdev = 0;
  RD_CUDA_CHECK(cudaGetDevice(&sdev));
  cudaStream_t st;
  if (sdev >= 0 && sdev < 64) {
    if (!s_st[sdev]) RD_CUDA_CHECK(cudaStreamCreateWithFlags(&s_st[sdev], cudaStreamNonBlocking));
    st = s_st[sdev];
  } else {
    RD_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  }
  const bool own_stream = !(sdev >= 0 && sdev < 64);
  // one workspace: A, BP, ring, stats, result, barrier (16-byte aligned pieces)
  const size_t bA = round_up(N * N * 2, 256), bBP = (size_t)(P / 2 * P * 4), bR = (size_t)((alpha_max + 1) * P * P * 2);
  const size_t bS = round_up((int64_t)(kmax + 1) * slen * 4, 256), bRes = round_up((6 + kmax + 1) * 4, 256);
  char *ws = nullptr;
  cudaError_t e = ws_malloc((void **)&ws, bA + bBP + bR + bS + bRes + 256, st);
  if (e != cudaSuccess) {
    if (own_stream) cudaStreamDestroy(st);
    (void)cudaGetLastError();
    return fail(RD_ENOMEM, "small_power_sequence: %s", cudaGetErrorString(e));
  }
  static thread_local int32_t *h_res = nullptr;
  static thread_local int h_cap = 0;
  if (h_cap < 6 + kmax + 1) {
    if (h_res) cudaFreeHost(h_res);
    h_res = nullptr;
    h_cap = 0;
    if (cudaMallocHost((void **)&h_res, (size_t)(6 + kmax + 1) * 4) != cudaSuccess) {
      h_res = nullptr;
      (void)cudaGetLastError();
      cudaFreeAsync(ws, st);
      if (own_stream) cudaStreamDestroy(st);
      return fail(RD_ENOMEM, "small_power_sequence: pinned result buffer");
    }
    h_cap = 6 + kmax + 1;
  }
  SmallArgs sa{};
  sa.A = reinterpret_cast<const int16_t *>(ws);
  sa.N = N; sa.P = P;
  sa.BP = reinterpret_cast<uint32_t *>(ws + bA);
  sa.ring = reinterpret_cast<int16_t *>(ws + bA + bBP);
  sa.stats = reinterpret_cast<int32_t *>(ws + bA + bBP + bR);
  sa.result = reinterpret_cast<int32_t *>(ws + bA + bBP + bR + bS);
  sa.bar = reinterpret_cast<unsigned *>(ws + bA + bBP + bR + bS + bRes);
  sa.kmax = kmax; sa.alpha_max = alpha_max; sa.policy = policy;
  int rc = RD_OK;
  // the upload is enqueued, not waited for (a pageable copy returns once the data is staged):
  // "build" ends here and the chain's time includes the copy's execution
  if ((e = cudaMemcpyAsync(ws, Ahost, (size_t)(N * N * 2), cudaMemcpyHostToDevice, st)) != cudaSuccess ||
      (e = cudaMemsetAsync(sa.bar, 0, 8, st)) != cudaSuccess)
    rc = fail(RD_ECUDA, "small_power_sequence: upload: %s", cudaGetErrorString(e));
  const auto t1 = std::chrono::steady_clock::now();
  if (rc == RD_OK) {
    // co-resident CTAs per device, queried once (the launch is cooperative: every CTA meets
    // the grid barrier); a one-tile order runs one CTA with an ordinary launch
    static int s_sms[64] = {}, s_per_sm[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    int sms = 148, per_sm = 1;
    if (dev >= 0 && dev < 64 && s_sms[dev]) {
      sms = s_sms[dev];
      per_sm = s_per_sm[dev];
    } else {
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, small_chain_kernel<false>, kSThreads, 0);
      if (dev >= 0 && dev < 64) { s_sms[dev] = sms; s_per_sm[dev] = per_sm; }
    }
    const int ntiles = (int)((P / kST) * (P / kST));
    const int grid = std::max(1, std::min(ntiles, sms * std::max(1, per_sm)));
    void *args[] = {&sa};
    if (grid == 1) {
      small_chain_kernel<true><<<1, kSThreads, 0, st>>>(sa);
      e = cudaGetLastError();
    } else {
      e = cudaLaunchCooperativeKernel((void *)small_chain_kernel<false>, grid, kSThreads, args, 0, st);
    }
    if (e != cudaSuccess ||
        (e = cudaMemcpyAsync(h_res, sa.result, (size_t)(6 + kmax + 1) * 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
      rc = fail(RD_ECUDA, "small_power_sequence: %s", cudaGetErrorString(e));
  }
  const auto t2 = std::chrono::steady_clock::now();
  cudaFreeAsync(ws, st);   // stream-ordered: the pool reuses it for the next call, no wait
  if (own_stream) {
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  }
  if (t_build) *t_build = std::chrono::duration<double>(t1 - t0).count();
  if (t_chain) *t_chain = std::chrono::duration<double>(t2 - t1).count();
  if (rc != RD_OK) return rc;
  const int k_stop = h_res[4];
  if (diag) {
    diag[1] = h_res[5];
    for (int k = 2; k <= k_stop; ++k) diag[k] = h_res[6 + k];
  }
  out->k_stop = k_stop;
  if (h_res[0]) {
    out->found = 1; out->n0 = h_res[1]; out->alpha = h_res[2]; out->beta = h_res[3];
    return RD_OK;
  }
  return RD_NOTFOUND;
}

}  // namespace rd
