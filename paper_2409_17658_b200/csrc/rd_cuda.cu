// Device half of librd.so (sm_100a): the (min,+) GEMM on DPX integer instructions with
// the fused diagonal-min / periodicity epilogue, the packing kernels, the power chain
// and the C-ABI entry points that touch the GPU.
//
// Paper: arXiv 2409.17658 (PAPER.md as P:<line>).  The operation is the (min,+) product
// c_ij = min_k (a_ik + b_kj) applied as A^{k+1} = A^k (x) A (Alg 2 step 3),
// with the diagonal min of Cor 7 and the test A^k = beta (x) A^{k-alpha} of
// Alg 2 step 4 / Prop 8 fused into the epilogue.
//
// Data layout: int16 entries, RD_INF = 0x3FFF = +inf.
//   pair-major ("PM") u32 layout of a matrix X used as the LEFT operand:
//       XT[t][i] = X[i][2t] | X[i][2t+1] << 16            (t = k-pair, i = row)
//   packed RIGHT operand:  BP[t][j] = B[2t][j] | B[2t+1][j] << 16
// Both are [K/2][rows-or-cols] u32 arrays, padded with INF to the CTA tile, so the
// mainloop needs no predicates: one VIADDMNMX.S16x2 computes min(x_lo + b_lo, acc_lo)
// and min(x_hi + b_hi, acc_hi) — two (min,+) terms (k = 2t and k = 2t+1) for one (i,j).
// The accumulators start at INF; min(lo, hi) in the epilogue finishes the k-reduction.
// The GEMM writes its output C = A^{k+1} directly in the PM layout (pairs along j), so
// the output of one power step is the left operand of the next one.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only; ranges cost nothing without an attached tool

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <vector>

#include "rd_internal.h"
#include "rd_gemm.cuh"

using namespace rd;

namespace rd {
// row-tiles per rasterisation group; measured at m = 9 (ncu DRAM read per launch): 8 -> 37.7 GB,
// 12 -> 41.3, 16 -> 47.4, 24 -> 68.5, 32 -> 85.8 GB, the same 276 ms
int g_raster_group = kGroup;
}  // namespace rd

// Scoped NVTX range (one per power step / chain build / power sequence)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Entry of every C-ABI call of this file: clear this thread's message and drop a stale,
// non-sticky CUDA error left by an earlier failed call (e.g. an out-of-memory cudaMalloc that
// was reported as RD_ENOMEM), so a later launch check does not report it again.
static inline void rd_enter() {
  clear_error();
  (void)cudaGetLastError();
}

namespace {

// ------------------------------------------------------------------ packing --
// Row-major int16 X (rows x cols, ld) -> PM u32 XT[cols_p/2][rows_p] (ld = rows_p).
// 32x32 u32 tile transpose through shared memory.  Entries > RD_INF clamp to RD_INF;
// everything outside (rows, cols) is INF.
__global__ void pack_left_kernel(const int16_t *__restrict__ X, int64_t ld, int64_t rows, int64_t cols,
                                 int64_t row0, uint32_t *__restrict__ XT, int64_t ldt, int64_t tpairs) {
  __shared__ uint32_t tile[32][33];
  const int64_t t0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int yy = ty; yy < 32; yy += 8) {
    int64_t i = i0 + yy, t = t0 + tx;
    uint32_t lo = RD_INF, hi = RD_INF;
    if (i < rows) {
      const int16_t *r = X + (row0 + i) * ld;
      int64_t k = 2 * t;
      if (k < cols) lo = (uint32_t)min((int)r[k], (int)RD_INF);
      if (k + 1 < cols) hi = (uint32_t)min((int)r[k + 1], (int)RD_INF);
    }
    tile[yy][tx] = lo | (hi << 16);
  }
  __syncthreads();
  for (int yy = ty; yy < 32; yy += 8) {
    int64_t t = t0 + yy, i = i0 + tx;
    if (t < tpairs && i < ldt) XT[t * ldt + i] = tile[tx][yy];
  }
}

// Row-major int16 B (K x N, ld) -> BP[t][j] = B[2t][j] | B[2t+1][j] << 16, padded with INF
// to (tpairs x ldp).
__global__ void pack_right_kernel(const int16_t *__restrict__ B, int64_t ld, int64_t K, int64_t N,
                                  uint32_t *__restrict__ BP, int64_t ldp, int64_t tpairs) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t t = blockIdx.y;
  if (j >= ldp || t >= tpairs) return;
  uint32_t lo = RD_INF, hi = RD_INF;
  if (j < N) {
    if (2 * t < K) lo = (uint32_t)min((int)B[(2 * t) * ld + j], (int)RD_INF);
    if (2 * t + 1 < K) hi = (uint32_t)min((int)B[(2 * t + 1) * ld + j], (int)RD_INF);
  }
  BP[t * ldp + j] = lo | (hi << 16);
}

// PM panel of rows [row0, row0+rows) of A from the packed right operand BP[t][j] =
// A[2t][j] | A[2t+1][j] << 16 (ld = ldp): XT[t][i] = A[row0+i][2t] | A[row0+i][2t+1] << 16.
__global__ void pm_from_bp_kernel(const uint32_t *__restrict__ BP, int64_t ldp, int64_t rows, int64_t row0,
                                  uint32_t *__restrict__ XT, int64_t ldt, int64_t tpairs) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, t = blockIdx.y;
  if (i >= ldt || t >= tpairs) return;
  uint32_t v = 0x3FFF3FFFu;
  if (i < rows) {
    const int64_t r = row0 + i;
    const uint32_t *src = BP + (r >> 1) * ldp;
    const int sh = (int)(r & 1) * 16;
    const uint32_t lo = (src[2 * t] >> sh) & 0xFFFF, hi = (src[2 * t + 1] >> sh) & 0xFFFF;
    v = lo | (hi << 16);
  }
  XT[t * ldt + i] = v;
}

// min over rows r in [r0, r1) of A[r][r] = half of BP[r/2][r] (INT_MAX if no finite one)
__global__ void diag_from_bp_kernel(const uint32_t *__restrict__ BP, int64_t ldp, int64_t r0, int64_t r1,
                                    int32_t *out) {
  const int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= r1) return;
  const int v = (int)((BP[(r >> 1) * ldp + r] >> ((r & 1) * 16)) & 0xFFFF);
  if (v < RD_INF) atomicMin(out, v);
}

// PM u32 XT[t][i] (ld = ldt) -> row-major int16 rows x cols (host-bound readback path).
__global__ void unpack_pm_kernel(const uint32_t *__restrict__ XT, int64_t ldt, int64_t rows, int64_t cols,
                                 int16_t *__restrict__ X) {
  int64_t i = blockIdx.y;
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows || k >= cols) return;
  uint32_t w = XT[(k >> 1) * ldt + i];
  X[i * cols + k] = (int16_t)((k & 1) ? (w >> 16) : (w & 0xFFFF));
}

__global__ void fill_u32_kernel(uint32_t *p, int64_t n, uint32_t v) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// MIN-reducible neutral stats: diag INT_MAX, lo INT_MAX, -hi INT_MAX, -mis 0, -fin 0.
__global__ void stats_init_kernel(int32_t *s, int alpha_max) {
  int i = threadIdx.x;
  int n = 1 + 4 * alpha_max;
  if (i >= n) return;
  int q = (i - 1) & 3;
  s[i] = (i == 0 || q == 0 || q == 1) ? INT_MAX : 0;
}

// Split-K combine for small grids: C = min over the nsplit partial PM tiles in W (HBM-bound,
// 16-byte accesses), written into the chain's ring slot, with the diagonal min and the
// periodicity stats of alphas [a0, a0 + 8) fused (pass a0 > 0 re-reads C instead of W).
// PM element e = t * ldc + i holds C[i][2t] | C[i][2t+1] << 16 (global row diag_row0 + i).
__global__ void __launch_bounds__(256) combine_pm_kernel(const uint32_t *__restrict__ W, int64_t stride, int nsplit,
                                                         uint32_t *__restrict__ C, int64_t nwords, int64_t ldc,
                                                         EpiArgs epi, int a0) {
  __shared__ int32_t red[8][1 + 4 * 8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int na = max(0, min(8, epi.nprev - a0));
  int32_t dmin = INT_MAX;
  uint32_t lo2[8], hi2[8], mis[8], fin[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) { lo2[a] = 0x7FFF7FFFu; hi2[a] = 0x80008000u; mis[a] = 0; fin[a] = 0; }
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nwords / 4; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = 4 * v;
    uint4 o;
    if (a0 == 0) {
      o = *reinterpret_cast<const uint4 *>(W + e);
      for (int sp = 1; sp < nsplit; ++sp) {
        const uint4 w = *reinterpret_cast<const uint4 *>(W + (int64_t)sp * stride + e);
        o.x = __vmins2(o.x, w.x); o.y = __vmins2(o.y, w.y); o.z = __vmins2(o.z, w.z); o.w = __vmins2(o.w, w.w);
      }
      *reinterpret_cast<uint4 *>(C + e) = o;
      // diagonal: row gi = diag_row0 + i meets column 2t or 2t + 1
      const int64_t t = e / ldc, i0 = e - t * ldc;
      const uint32_t ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t gi = epi.diag_row0 + i0 + q;
        if (gi == 2 * t) dmin = min(dmin, (int)(ow[q] & 0xFFFF));
        if (gi == 2 * t + 1) dmin = min(dmin, (int)(ow[q] >> 16));
      }
    } else {
      o = *reinterpret_cast<const uint4 *>(C + e);
    }
    const uint32_t ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      if (a < na) {
        const uint4 pv = *reinterpret_cast<const uint4 *>(epi.prev[a0 + a] + e);
        const uint32_t pw[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) stats_pair(ow[q], pw[q], lo2[a], hi2[a], mis[a], fin[a]);
      }
    }
  }
  dmin = __reduce_min_sync(0xffffffffu, dmin);
  if (lane == 0) red[warp][0] = dmin;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    int32_t lo = min((int32_t)(int16_t)(lo2[a] & 0xFFFF), (int32_t)(int16_t)(lo2[a] >> 16));
    int32_t hi = max((int32_t)(int16_t)(hi2[a] & 0xFFFF), (int32_t)(int16_t)(hi2[a] >> 16));
    if (!fin[a]) { lo = INT_MAX; hi = INT_MIN + 1; }
    int32_t v0 = __reduce_min_sync(0xffffffffu, lo);
    int32_t v1 = __reduce_min_sync(0xffffffffu, -hi);
    int32_t v2 = __reduce_min_sync(0xffffffffu, mis[a] ? -1 : 0);
    int32_t v3 = __reduce_min_sync(0xffffffffu, fin[a] ? -1 : 0);
    if (lane == 0) {
      red[warp][1 + 4 * a] = v0; red[warp][2 + 4 * a] = v1; red[warp][3 + 4 * a] = v2; red[warp][4 + 4 * a] = v3;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 1 + 4 * na; e += blockDim.x) {
    int32_t v = red[0][e];
    for (int w = 1; w < 8; ++w) v = min(v, red[w][e]);
    if (e == 0) {
      if (a0 == 0) atomicMin(epi.stats, v);
    } else {
      atomicMin(epi.stats + 4 * a0 + e, v);
    }
  }
}

int g_dpx_cols = 3;       // rd_set_gemm_variant (default: measured best)
int g_dpx_auto = 1;       // long dense chain steps tune 3 vs 4 per chain until rd_set_gemm_variant is called
int g_gemm_tile = 0;      // rd_set_gemm_tile: 0 = the chain's wave model picks, 64 / 128 forced
int g_sparse_bytes = 2;   // rd_set_sparse_bytes: 0 16-bit kernel, 1 byte kernel, 2 slab byte kernel

__global__ void pack_t32_kernel(const int32_t *__restrict__ X, int64_t ld, int64_t rows, int64_t cols,
                                int32_t *__restrict__ XT, int64_t ldt, int64_t kp) {
  __shared__ int32_t tile[32][33];
  const int64_t k0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int yy = ty; yy < 32; yy += 8) {
    const int64_t i = i0 + yy, k = k0 + tx;
    tile[yy][tx] = (i < rows && k < cols) ? min(X[i * ld + k], kInf32) : kInf32;
  }
  __syncthreads();
  for (int yy = ty; yy < 32; yy += 8) {
    const int64_t k = k0 + yy, i = i0 + tx;
    if (k < kp && i < ldt) XT[k * ldt + i] = tile[tx][yy];
  }
}

__global__ void pack_copy32_kernel(const int32_t *__restrict__ B, int64_t ld, int64_t K, int64_t N,
                                   int32_t *__restrict__ BP, int64_t ldp, int64_t kp) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, k = blockIdx.y;
  if (j >= ldp || k >= kp) return;
  BP[k * ldp + j] = (j < N && k < K) ? min(B[k * ld + j], kInf32) : kInf32;
}


template <bool OUT_PM, bool STATS>
int launch_gemm(const uint32_t *XT, int64_t ldx, const uint32_t *BP, int64_t ldb, int64_t kpairs, void *C,
                int64_t ldc, int64_t M, int64_t N, int64_t Mp, int64_t Np, const EpiArgs &epi,
                cudaStream_t st, int nsplit = 1, const TmaOps *tma = nullptr, int tn = 128, int dpx = -1) {
  const PeerB pb{};
  const int dcols = dpx >= 0 ? dpx : g_dpx_cols;
  if (OUT_PM && STATS && epi.sk_nsk > 0) {   // stream-K step (rd_set_stream_k)
#define RD_LGS(D, T) launch_gemm_v<kOutPM, true, D, T, true>(XT, ldx, BP, ldb, kpairs, C, ldc, M, N, Mp, Np, epi, st, 1, pb, tma)
#define RD_LGS2(D) return tma ? RD_LGS(D, true) : RD_LGS(D, false)
    switch (dcols) {
      case 0: RD_LGS2(0);
      case 2: RD_LGS2(2);
      case 3: RD_LGS2(3);
      case 4: RD_LGS2(4);
      default: RD_LGS2(8);
    }
#undef RD_LGS2
#undef RD_LGS
  }
  if (OUT_PM && tma) {   // the chain's PM step with the TMA mainloop (rd_set_gemm_tma)
#define RD_LGT(D) launch_gemm_v<kOutPM, STATS, D, true>(XT, ldx, BP, ldb, kpairs, C, ldc, M, N, Mp, Np, epi, st, nsplit, pb, tma)
    switch (dcols) {
      case 0: return RD_LGT(0);
      case 2: return RD_LGT(2);
      case 3: return RD_LGT(3);
      case 4: return RD_LGT(4);
      default: return RD_LGT(8);
    }
#undef RD_LGT
  }
  if (OUT_PM && tn == 64 && !tma) {   // 128 x 64 tiles, 3 CTAs per SM (the chain's wave model)
#define RD_LG64(D) launch_gemm_v<kOutPM, STATS, D, false, false, 64>(XT, ldx, BP, ldb, kpairs, C, ldc, M, N, Mp, Np, epi, st, nsplit, pb)
    switch (dcols) {
      case 0: return RD_LG64(0);
      case 2: return RD_LG64(2);
      case 3: return RD_LG64(3);
      case 4: return RD_LG64(4);
      default: return RD_LG64(8);
    }
#undef RD_LG64
  }
#define RD_LG(D) launch_gemm_v<OUT_PM ? kOutPM : kOutRow, STATS, D>(XT, ldx, BP, ldb, kpairs, C, ldc, M, N, Mp, Np, epi, st, nsplit, pb)
  switch (dcols) {
    case 0: return RD_LG(0);
    case 2: return RD_LG(2);
    case 3: return RD_LG(3);
    case 4: return RD_LG(4);
    default: return RD_LG(8);
  }
#undef RD_LG
}

int launch_gemm32(const int32_t *XT, int64_t ldx, const int32_t *BP, int64_t ldb, int64_t kp, int32_t *C,
                  int64_t ldc, int64_t M, int64_t N, int64_t Mp, int64_t Np, int accumulate, cudaStream_t st) {
#define RD_LG32(D) launch_gemm32_v<D>(XT, ldx, BP, ldb, kp, C, ldc, M, N, Mp, Np, accumulate, st)
  switch (g_dpx_cols) {
    case 0: return RD_LG32(0);
    case 2: return RD_LG32(2);
    case 3: return RD_LG32(3);
    case 4: return RD_LG32(4);
    default: return RD_LG32(8);
  }
#undef RD_LG32
}

int pack_left(const int16_t *X, int64_t ld, int64_t rows, int64_t cols, int64_t row0, uint32_t *XT,
              int64_t ldt, int64_t tpairs, cudaStream_t st) {
  dim3 grid((unsigned)((tpairs + 31) / 32), (unsigned)((ldt + 31) / 32));
  pack_left_kernel<<<grid, dim3(32, 8), 0, st>>>(X, ld, rows, cols, row0, XT, ldt, tpairs);
  RD_CUDA_CHECK(cudaGetLastError());
  return RD_OK;
}

int pack_right(const int16_t *B, int64_t ld, int64_t K, int64_t N, uint32_t *BP, int64_t ldp, int64_t tpairs,
               cudaStream_t st) {
  dim3 grid((unsigned)((ldp + 255) / 256), (unsigned)tpairs);
  pack_right_kernel<<<grid, 256, 0, st>>>(B, ld, K, N, BP, ldp, tpairs);
  RD_CUDA_CHECK(cudaGetLastError());
  return RD_OK;
}

}  // namespace

extern "C" int rd_set_gemm_variant(int dpx_cols) try {
  rd_enter();
  if (dpx_cols == -1) {   // back to the default: 3, tuned per long chain
    g_dpx_cols = 3;
    g_dpx_auto = 1;
    return RD_OK;
  }
  if (dpx_cols != 0 && dpx_cols != 2 && dpx_cols != 3 && dpx_cols != 4 && dpx_cols != 8)
    return fail(RD_EINVAL, "rd_set_gemm_variant: dpx_cols must be one of -1 (auto), 0, 2, 3, 4, 8");
  g_dpx_cols = dpx_cols;
  g_dpx_auto = 0;   // an explicit choice: no per-chain tuning
  return RD_OK;
} RD_ABI_CATCH("rd_set_gemm_variant")

extern "C" int rd_set_gemm_tile(int tn) try {
  rd_enter();
  if (tn != 0 && tn != 64 && tn != 128) return fail(RD_EINVAL, "rd_set_gemm_tile: 0 (model), 64 or 128");
  g_gemm_tile = tn;
  return RD_OK;
} RD_ABI_CATCH("rd_set_gemm_tile")

extern "C" int rd_set_device(int device) try {
  rd_enter();
  RD_CUDA_CHECK(cudaSetDevice(device));
  return RD_OK;
} RD_ABI_CATCH("rd_set_device")

// =========================================================== generic product ==
// Library-owned stream-ordered pool (one per device; chains and the generic products' workspace).
namespace rd {
constexpr uint64_t kPoolKeep = (uint64_t)16 << 30;
constexpr size_t kPoolMax = (size_t)kPoolKeep;
cudaMemPool_t chain_pool(int dev) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&pools[dev], &props) != cudaSuccess) {
      (void)cudaGetLastError();
      pools[dev] = nullptr;
      return nullptr;
    }
    uint64_t thr = kPoolKeep;
    cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
  }
  return pools[dev];
}

// Stream-ordered workspace from the library's pool (the device's default pool and its release
// threshold are left alone: other cudaMallocAsync users in the process keep their setting);
// falls back to cudaMallocAsync on the default pool if the library pool cannot be created.
cudaError_t ws_malloc(void **p, size_t bytes, cudaStream_t st) {
  *p = nullptr;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (cudaMemPool_t pool = chain_pool(dev)) {
    if ((e = cudaMallocFromPoolAsync(p, bytes, pool, st)) == cudaSuccess) return e;
    (void)cudaGetLastError();
    *p = nullptr;
  }
  return cudaMallocAsync(p, bytes, st);
}
}  // namespace rd

static int minplus_rowmajor(const int16_t *A, int64_t lda, const int16_t *B, int64_t ldb, int16_t *C,
                            int64_t ldc, int64_t M, int64_t N, int64_t K, void *cuda_stream, int accumulate,
                            const char *who) {
  rd_enter();
  if (!A || !B || !C) return fail(RD_EINVAL, "%s: NULL pointer", who);
  if (M < 1 || N < 1 || K < 1) return fail(RD_EINVAL, "%s: M, N, K must be >= 1", who);
  if (lda < K || ldb < N || ldc < N) return fail(RD_EINVAL, "%s: leading dimension too small", who);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int64_t Mp = round_up(M, kTile), Np = round_up(N, kTile), Kp = round_up(K, 2 * kBK2);
  const int64_t kpairs = Kp / 2;
  uint32_t *XT = nullptr, *BP = nullptr;
  cudaError_t e = ws_malloc((void **)&XT, (size_t)(kpairs * Mp * 4), st);
  if (e == cudaSuccess) e = ws_malloc((void **)&BP, (size_t)(kpairs * Np * 4), st);
  if (e != cudaSuccess) {
    if (XT) cudaFreeAsync(XT, st);
    (void)cudaGetLastError();
    return fail(RD_ENOMEM, "%s: workspace: %s", who, cudaGetErrorString(e));
  }
  int rc = pack_left(A, lda, M, K, 0, XT, Mp, kpairs, st);
  if (rc == RD_OK) rc = pack_right(B, ldb, K, N, BP, Np, kpairs, st);
  EpiArgs epi{};
  epi.accumulate = accumulate;
  if (rc == RD_OK) rc = launch_gemm<false, false>(XT, Mp, BP, Np, kpairs, C, ldc, M, N, Mp, Np, epi, st);
  cudaFreeAsync(XT, st);
  cudaFreeAsync(BP, st);
  return rc;
}

extern "C" int rd_minplus_mul_ex(const int16_t *A, int64_t lda, const int16_t *B, int64_t ldb, int16_t *C,
                                 int64_t ldc, int64_t M, int64_t N, int64_t K, void *cuda_stream) try {
  return minplus_rowmajor(A, lda, B, ldb, C, ldc, M, N, K, cuda_stream, 0, "rd_minplus_mul_ex");
} RD_ABI_CATCH("rd_minplus_mul_ex")

extern "C" int rd_minplus_mul_acc(const int16_t *A, int64_t lda, const int16_t *B, int64_t ldb, int16_t *C,
                                  int64_t ldc, int64_t M, int64_t N, int64_t K, void *cuda_stream) try {
  return minplus_rowmajor(A, lda, B, ldb, C, ldc, M, N, K, cuda_stream, 1, "rd_minplus_mul_acc");
} RD_ABI_CATCH("rd_minplus_mul_acc")

static int minplus32_rowmajor(const int32_t *A, int64_t lda, const int32_t *B, int64_t ldb, int32_t *C,
                              int64_t ldc, int64_t M, int64_t N, int64_t K, void *cuda_stream, const char *who) {
  rd_enter();
  if (!A || !B || !C) return fail(RD_EINVAL, "%s: NULL pointer", who);
  if (M < 1 || N < 1 || K < 1) return fail(RD_EINVAL, "%s: M, N, K must be >= 1", who);
  if (lda < K || ldb < N || ldc < N) return fail(RD_EINVAL, "%s: leading dimension too small", who);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int64_t Mp = round_up(M, kTile), Np = round_up(N, kTile), Kp = round_up(K, kBK2);
  int32_t *XT = nullptr, *BP = nullptr;
  cudaError_t e = ws_malloc((void **)&XT, (size_t)(Kp * Mp * 4), st);
  if (e == cudaSuccess) e = ws_malloc((void **)&BP, (size_t)(Kp * Np * 4), st);
  if (e != cudaSuccess) {
    if (XT) cudaFreeAsync(XT, st);
    (void)cudaGetLastError();
    return fail(RD_ENOMEM, "%s: workspace: %s", who, cudaGetErrorString(e));
  }
  pack_t32_kernel<<<dim3((unsigned)((Kp + 31) / 32), (unsigned)((Mp + 31) / 32)), dim3(32, 8), 0, st>>>(
      A, lda, M, K, XT, Mp, Kp);
  pack_copy32_kernel<<<dim3((unsigned)((Np + 255) / 256), (unsigned)Kp), 256, 0, st>>>(B, ldb, K, N, BP, Np, Kp);
  int rc = RD_OK;
  if ((e = cudaGetLastError()) != cudaSuccess) rc = fail(RD_ECUDA, "%s: %s", who, cudaGetErrorString(e));
  if (rc == RD_OK) rc = launch_gemm32(XT, Mp, BP, Np, Kp, C, ldc, M, N, Mp, Np, 0, st);
  cudaFreeAsync(XT, st);
  cudaFreeAsync(BP, st);
  return rc;
}

extern "C" int rd_minplus_mul32_ex(const int32_t *A, int64_t lda, const int32_t *B, int64_t ldb, int32_t *C,
                                   int64_t ldc, int64_t M, int64_t N, int64_t K, void *cuda_stream) try {
  return minplus32_rowmajor(A, lda, B, ldb, C, ldc, M, N, K, cuda_stream, "rd_minplus_mul32_ex");
} RD_ABI_CATCH("rd_minplus_mul32_ex")

extern "C" int rd_minplus_mul32(const int32_t *A, const int32_t *B, int32_t *C, int64_t N) try {
  return minplus32_rowmajor(A, N, B, N, C, N, N, N, N, nullptr, "rd_minplus_mul32");
} RD_ABI_CATCH("rd_minplus_mul32")

// ------------------------------------------------------- standalone stats --
// Stats of a row-major int16 panel `cur` (rows x cols, ld) against up to kMaxAlpha
// earlier panels of the same shape, in the MIN-reducible layout of rd_chain_step
// (the standalone form of the fused epilogue; HBM-bound).
struct PanelStatsArgs {
  const int16_t *prev[kMaxAlpha];
  int nprev;
};

// Single pass over every alpha in [a0, a0 + NA): a thread holds one 16-byte chunk of the
// current power (8 entries) in registers, loads the same chunk of each earlier power once and
// folds it into that alpha's packed (lo, -hi, mis, fin) registers; the block reduces at the
// end.  HBM bytes (1 + nprev) * 2 * rows * cols, each read exactly once.
// NA = the number of alphas of this pass exactly (0: diagonal only), so every load is
// unconditional and all 1 + NA chunks of a thread are in flight together.
template <int NA>
__global__ void __launch_bounds__(256) panel_stats_kernel(const int16_t *__restrict__ cur, int64_t rows,
                                                          int64_t cols, int64_t ld, int64_t diag_row0,
                                                          PanelStatsArgs pa, int a0, int32_t *__restrict__ stats) {
  constexpr int NR = NA > 0 ? NA : 1;
  __shared__ int32_t red[8][1 + 4 * NR];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int na = NA;
  int32_t dmin = INT_MAX;
  uint32_t lo2[NR], hi2[NR], mis[NR], fin[NR];
#pragma unroll
  for (int a = 0; a < NR; ++a) { lo2[a] = 0x7FFF7FFFu; hi2[a] = 0x80008000u; mis[a] = 0; fin[a] = 0; }
  // the earlier powers' base pointers in registers (not re-read from the parameter block)
  const int16_t *pp[NR];
  bool vec = (ld % 8 == 0) && ((reinterpret_cast<uintptr_t>(cur) & 15) == 0);
#pragma unroll
  for (int a = 0; a < NA; ++a) {
    pp[a] = pa.prev[a0 + a];
    vec = vec && ((reinterpret_cast<uintptr_t>(pp[a]) & 15) == 0);
  }
  const int64_t cpr = (cols + 7) / 8, total = rows * cpr;
  auto scalar8 = [&](const int16_t *base, int64_t off, int64_t j, uint32_t (&w)[4]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool in0 = j + 2 * q < cols, in1 = j + 2 * q + 1 < cols;
      w[q] = (in0 ? (uint16_t)base[off + 2 * q] : (uint16_t)RD_INF) |
             ((uint32_t)(in1 ? (uint16_t)base[off + 2 * q + 1] : (uint16_t)RD_INF) << 16);
    }
  };
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < total; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = v / cpr, j = (v - i * cpr) * 8;
    const int64_t off = i * ld + j;
    uint32_t o[4], w[NR][4];
    if (vec && j + 8 <= cols) {
      // fast path: all 1 + NA 16-byte loads issued before any is used
      const uint4 x = __ldcs(reinterpret_cast<const uint4 *>(cur + off));
      uint4 y[NR];
#pragma unroll
      for (int a = 0; a < NA; ++a) y[a] = __ldcs(reinterpret_cast<const uint4 *>(pp[a] + off));
      o[0] = x.x; o[1] = x.y; o[2] = x.z; o[3] = x.w;
#pragma unroll
      for (int a = 0; a < NA; ++a) { w[a][0] = y[a].x; w[a][1] = y[a].y; w[a][2] = y[a].z; w[a][3] = y[a].w; }
    } else {
      scalar8(cur, off, j, o);
#pragma unroll
      for (int a = 0; a < NA; ++a) scalar8(pp[a], off, j, w[a]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = __vminu2(o[q], kInf2);   // entries above RD_INF read as +inf
    if (a0 == 0) {   // diagonal (Cor 7): global row diag_row0 + i meets column j .. j + 7
      const int64_t gi = diag_row0 + i;
      if (gi >= j && gi < j + 8) {
        const int t = (int)(gi - j);
        dmin = min(dmin, (int)((o[t >> 1] >> (16 * (t & 1))) & 0xFFFF));
      }
    }
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q) stats_pair(o[q], __vminu2(w[a][q], kInf2), lo2[a], hi2[a], mis[a], fin[a]);
  }
  dmin = __reduce_min_sync(0xffffffffu, dmin);
  if (lane == 0) red[warp][0] = dmin;
#pragma unroll
  for (int a = 0; a < NA; ++a) {
    int32_t lo = min((int32_t)(int16_t)(lo2[a] & 0xFFFF), (int32_t)(int16_t)(lo2[a] >> 16));
    int32_t hi = max((int32_t)(int16_t)(hi2[a] & 0xFFFF), (int32_t)(int16_t)(hi2[a] >> 16));
    if (!(fin[a] & 0xFFFF) && !(fin[a] >> 16)) { lo = INT_MAX; hi = INT_MIN + 1; }
    const int32_t v0 = __reduce_min_sync(0xffffffffu, lo), v1 = __reduce_min_sync(0xffffffffu, -hi);
    const int32_t v2 = __reduce_min_sync(0xffffffffu, mis[a] ? -1 : 0);
    const int32_t v3 = __reduce_min_sync(0xffffffffu, fin[a] ? -1 : 0);
    if (lane == 0) {
      red[warp][1 + 4 * a] = v0; red[warp][2 + 4 * a] = v1; red[warp][3 + 4 * a] = v2; red[warp][4 + 4 * a] = v3;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 1 + 4 * na; e += blockDim.x) {
    int32_t v = red[0][e];
#pragma unroll
    for (int w2 = 1; w2 < 8; ++w2) v = min(v, red[w2][e]);
    if (e == 0) {
      if (a0 == 0) atomicMin(stats, v);
    } else {
      atomicMin(stats + 4 * a0 + e, v);
    }
  }
}

// Streaming form of panel_stats_kernel for 16-byte aligned panels (ld % 8 == 0): every thread
// keeps PS stages of its chunks (the current power's and each earlier power's 16 bytes) in
// flight with cp.async into its own shared-memory slots — no registers held by outstanding
// loads, so one 256-thread block per SM sustains ~PS x 45 KB in flight — and folds a stage
// once it lands.  A ragged last chunk of a row is zero-filled by cp.async and re-marked +inf.
__device__ __forceinline__ void cp_async16_zfill(void *smem, const void *gmem, int bytes) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(bytes));
}

template <int NA, int PS, int T>
__global__ void __launch_bounds__(T, 1) panel_stats_stream_kernel(const int16_t *__restrict__ cur, int64_t rows,
                                                                int64_t cols, int64_t ld, int64_t diag_row0,
                                                                PanelStatsArgs pa, int a0, int32_t *__restrict__ stats) {
  constexpr int NR = NA > 0 ? NA : 1, NW = T / 32;
  extern __shared__ uint4 sbuf[];   // [PS][1 + NA][T]
  __shared__ int32_t red[NW][1 + 4 * NR];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int32_t dmin = INT_MAX;
  uint32_t lo2[NR], hi2[NR], mis[NR], fin[NR];
#pragma unroll
  for (int a = 0; a < NR; ++a) { lo2[a] = 0x7FFF7FFFu; hi2[a] = 0x80008000u; mis[a] = 0; fin[a] = 0; }
  const int16_t *pp[NR];
#pragma unroll
  for (int a = 0; a < NA; ++a) pp[a] = pa.prev[a0 + a];
  // chunk v = (row i, column chunk jc); a thread walks v = v0, v0 + gs, ... with (i, jc) kept
  // incrementally (no divisions in the loop): one cursor for the loads, one for the folds
  const int64_t cpr = (cols + 7) / 8, total = rows * cpr;
  const int64_t gs = (int64_t)gridDim.x * T, v0 = (int64_t)blockIdx.x * T + tid;
  const int64_t gs_q = gs / cpr, gs_r = gs - gs_q * cpr;
  struct Cursor {
    int64_t v, i, jc;
  };
  auto advance = [&](Cursor &c) {
    c.v += gs;
    c.i += gs_q;
    c.jc += gs_r;
    if (c.jc >= cpr) { c.jc -= cpr; ++c.i; }
  };
  Cursor ld_c{v0, v0 / cpr, v0 - (v0 / cpr) * cpr}, cs = ld_c;
  auto slot = [&](int st, int arr) -> uint4 * { return &sbuf[(st * (1 + NA) + arr) * T + tid]; };
  auto issue = [&](int st) {
    if (ld_c.v < total) {
      const int64_t j = ld_c.jc * 8, off = ld_c.i * ld + j;
      const int bytes = j + 8 <= cols ? 16 : (int)(cols - j) * 2;
      cp_async16_zfill(slot(st, 0), cur + off, bytes);
#pragma unroll
      for (int a = 0; a < NA; ++a) cp_async16_zfill(slot(st, 1 + a), pp[a] + off, bytes);
    }
    cp_async_commit();
    advance(ld_c);
  };
#pragma unroll
  for (int st = 0; st < PS - 1; ++st) issue(st);
  int st_ld = PS - 1, st = 0;
  for (; cs.v < total; advance(cs)) {
    issue(st_ld);
    st_ld = st_ld + 1 == PS ? 0 : st_ld + 1;
    cp_async_wait<PS - 1>();
    const int64_t j = cs.jc * 8;
    // lanes past the row's end (zero-filled) become +inf in both powers: neutral in the stats
    const uint4 x = *slot(st, 0);
    uint32_t o[4] = {x.x, x.y, x.z, x.w};
    uint32_t padw[4] = {0, 0, 0, 0};
    if (j + 8 > cols) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        padw[q] = (j + 2 * q < cols ? 0u : 0x0000FFFFu) | (j + 2 * q + 1 < cols ? 0u : 0xFFFF0000u);
    }
    uint32_t io = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      o[q] = __vminu2(o[q] | padw[q], kInf2);
      io |= __vcmpeq2(o[q], kInf2);
    }
    if (a0 == 0) {
      const int64_t gi = diag_row0 + cs.i;
      if (gi >= j && gi < j + 8 && gi < cols) {
        const int t = (int)(gi - j);
        dmin = min(dmin, (int)((o[t >> 1] >> (16 * (t & 1))) & 0xFFFF));
      }
    }
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      const uint4 y = *slot(st, 1 + a);
      uint32_t w[4] = {y.x, y.y, y.z, y.w};
      uint32_t iw = io;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        w[q] = __vminu2(w[q] | padw[q], kInf2);
        iw |= __vcmpeq2(w[q], kInf2);
      }
      if (iw == 0) {   // every lane finite in both powers (every entry from k = 4 on)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t d = __vsub2(o[q], w[q]);
          lo2[a] = __vmins2(lo2[a], d);
          hi2[a] = __vmaxs2(hi2[a], d);
        }
        fin[a] = 0xFFFFFFFFu;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) stats_pair(o[q], w[q], lo2[a], hi2[a], mis[a], fin[a]);
      }
    }
    st = st + 1 == PS ? 0 : st + 1;
  }
  cp_async_wait<0>();
  dmin = __reduce_min_sync(0xffffffffu, dmin);
  if (lane == 0) red[warp][0] = dmin;
#pragma unroll
  for (int a = 0; a < NA; ++a) {
    int32_t lo = min((int32_t)(int16_t)(lo2[a] & 0xFFFF), (int32_t)(int16_t)(lo2[a] >> 16));
    int32_t hi = max((int32_t)(int16_t)(hi2[a] & 0xFFFF), (int32_t)(int16_t)(hi2[a] >> 16));
    if (!(fin[a] & 0xFFFF) && !(fin[a] >> 16)) { lo = INT_MAX; hi = INT_MIN + 1; }
    const int32_t v0r = __reduce_min_sync(0xffffffffu, lo), v1 = __reduce_min_sync(0xffffffffu, -hi);
    const int32_t v2 = __reduce_min_sync(0xffffffffu, mis[a] ? -1 : 0);
    const int32_t v3 = __reduce_min_sync(0xffffffffu, fin[a] ? -1 : 0);
    if (lane == 0) {
      red[warp][1 + 4 * a] = v0r; red[warp][2 + 4 * a] = v1; red[warp][3 + 4 * a] = v2; red[warp][4 + 4 * a] = v3;
    }
  }
  __syncthreads();
  for (int e = tid; e < 1 + 4 * NA; e += T) {
    int32_t v = red[0][e];
#pragma unroll
    for (int w2 = 1; w2 < NW; ++w2) v = min(v, red[w2][e]);
    if (e == 0) {
      if (a0 == 0) atomicMin(stats, v);
    } else {
      atomicMin(stats + 4 * a0 + e, v);
    }
  }
}

// Diagonal min (Cor 7) of a row panel: row i meets column diag_row0 + i (for the flat form of
// the streaming kernel, which sees the panel as one contiguous array).
__global__ void panel_diag_kernel(const int16_t *__restrict__ cur, int64_t rows, int64_t cols, int64_t ld,
                                  int64_t diag_row0, int32_t *__restrict__ stats) {
  int32_t v = INT_MAX;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = diag_row0 + i;
    if (c >= 0 && c < cols) v = min(v, min((int)cur[i * ld + c], (int)RD_INF));
  }
  v = __reduce_min_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && v != INT_MAX) atomicMin(stats, v);
}

template <int NA>
static int launch_panel_stats(const int16_t *cur, int64_t rows, int64_t cols, int64_t ld, int64_t diag_row0,
                              const PanelStatsArgs &pa, int a0, int32_t *stats, int sms, cudaStream_t st, bool vec,
                              bool flat) {
  if (flat) {
    // a contiguous panel (ld == cols) with 16-byte aligned bases is one flat array of rows x cols
    // entries: stream it in aligned 16-byte chunks whatever cols is (the stats are elementwise;
    // the diagonal goes to panel_diag_kernel)
    if (a0 == 0) {
      panel_diag_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((rows + 255) / 256, 4 * sms)), 256, 0,
                          st>>>(cur, rows, cols, ld, diag_row0, stats);
      RD_CUDA_CHECK(cudaGetLastError());
    }
    cols = rows * cols;
    ld = cols;
    rows = 1;
    diag_row0 = INT64_MIN / 2;   // no element meets the "diagonal" of the flat view
    vec = true;
  }
  const int64_t chunks = rows * ((cols + 7) / 8);
  if (vec) {
    // 512 threads (16 warps) and 2-4 stages while the stage buffers fit 200 KB; 256 threads and
    // 3 stages for the widest passes
    constexpr int T = (1 + NA) * 8192 * 2 <= 200 * 1024 ? 512 : 256;
    constexpr int PS0 = (220 * 1024) / ((1 + NA) * 16 * T);
    constexpr int PS = PS0 > 4 ? 4 : (PS0 < 2 ? 2 : PS0);
    constexpr int smem = PS * (1 + NA) * 16 * T;
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !attr[dev]) {
      RD_CUDA_CHECK(cudaFuncSetAttribute(panel_stats_stream_kernel<NA, PS, T>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attr[dev] = true;
    }
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((chunks + T - 1) / T, (int64_t)sms));
    panel_stats_stream_kernel<NA, PS, T><<<grid, T, smem, st>>>(cur, rows, cols, ld, diag_row0, pa, a0, stats);
  } else {
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((chunks + 255) / 256, (int64_t)sms * 4));
    panel_stats_kernel<NA><<<grid, 256, 0, st>>>(cur, rows, cols, ld, diag_row0, pa, a0, stats);
  }
  RD_CUDA_CHECK(cudaGetLastError());
  return RD_OK;
}

extern "C" int rd_panel_stats(const int16_t *cur, const int16_t *const *prev, int nprev, int64_t rows,
                              int64_t cols, int64_t ld, int64_t diag_row0, int alpha_max, int32_t *stats_dev,
                              void *cuda_stream) try {
  rd_enter();
  if (!cur || !stats_dev || (nprev > 0 && !prev)) return fail(RD_EINVAL, "rd_panel_stats: NULL argument");
  if (alpha_max < 1 || alpha_max > kMaxAlpha || nprev < 0 || nprev > alpha_max)
    return fail(RD_EINVAL, "rd_panel_stats: need 0 <= nprev <= alpha_max <= 32");
  if (rows < 0 || cols < 1 || ld < cols) return fail(RD_EINVAL, "rd_panel_stats: bad shape");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  PanelStatsArgs pa{};
  pa.nprev = nprev;
  for (int a = 0; a < nprev; ++a) {
    if (!prev[a]) return fail(RD_EINVAL, "rd_panel_stats: prev[%d] is NULL", a);
    pa.prev[a] = prev[a];
  }
  stats_init_kernel<<<1, 1 + 4 * kMaxAlpha, 0, st>>>(stats_dev, alpha_max);
  RD_CUDA_CHECK(cudaGetLastError());
  if (rows == 0) return RD_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one thread per 16-byte chunk of the panel, grid-strided; every alpha of a pass in one sweep
  // (16-byte aligned panels: the cp.async streaming kernel, one block per SM)
  bool aligned = (reinterpret_cast<uintptr_t>(cur) & 15) == 0;
  for (int a = 0; a < nprev; ++a) aligned = aligned && ((reinterpret_cast<uintptr_t>(pa.prev[a]) & 15) == 0);
  const bool vec = aligned && (ld % 8 == 0), flat = aligned && ld == cols && !vec;
  for (int a0 = 0; a0 < std::max(nprev, 1); a0 += 16) {
    const int na = std::min(16, nprev - a0);
    int rc = RD_OK;
    switch (na) {
#define RD_PS(K) \
  case K: rc = launch_panel_stats<K>(cur, rows, cols, ld, diag_row0, pa, a0, stats_dev, sms, st, vec, flat); break;
      RD_PS(0) RD_PS(1) RD_PS(2) RD_PS(3) RD_PS(4) RD_PS(5) RD_PS(6) RD_PS(7) RD_PS(8)
      RD_PS(9) RD_PS(10) RD_PS(11) RD_PS(12) RD_PS(13) RD_PS(14) RD_PS(15) RD_PS(16)
#undef RD_PS
    }
    if (rc != RD_OK) return rc;
  }
  return RD_OK;
} RD_ABI_CATCH("rd_panel_stats")

extern "C" int rd_minplus_mul(const int16_t *A, const int16_t *B, int16_t *C, int64_t N) try {
  if (!A || !B || !C) { rd_enter(); return fail(RD_EINVAL, "rd_minplus_mul: NULL pointer"); }
  if (N < 1) { rd_enter(); return fail(RD_EINVAL, "rd_minplus_mul: N must be >= 1"); }
  if (C == A || C == B) { rd_enter(); return fail(RD_EINVAL, "rd_minplus_mul: C aliases an input"); }
  return rd_minplus_mul_ex(A, N, B, N, C, N, N, N, N, nullptr);
} RD_ABI_CATCH("rd_minplus_mul")

namespace {
// ======================================================= structured step ==
// NEXT-3: the right operand of every power step is the fixed, sparse A(G)
// (0.55% dense at m = 9), so C[i][j] = min_{q : A[q][j] finite} (X[i][q] + A[q][j]) — the
// same (min,+) product with the infinite terms skipped, N * nnz(A) terms per
// step instead of N^3.  Layout "RP" (row pairs): RP[p][j] = X[2p][j] | X[2p+1][j] << 16.
// One CTA owns 4 rows (2 row pairs); the q-range of those rows is staged in shared memory
// as uint2 (both pairs of one q), chunked when N * 8 B exceeds shared memory.  A warp
// takes one output column at a time: its lanes split the column's CSC entries
// (q, w), each lane gathers xs[q] and applies two VIADDMNMX.S16x2 (4 rows), and a
// butterfly of VIMNMX folds the lanes.  The diagonal min and the per-alpha periodicity
// stats are fused (lane a owns alpha a+1), as in the dense epilogue.
struct SpArgs {
  const int32_t *colptr;  // nchunks x (N + 1) absolute offsets into ent
  const uint32_t *ent;    // general: (q - chunk start) | w << 17;  uniform: (q - chunk start) * 8
  int nchunks, Qc;
  int64_t N;              // columns
  const int16_t *wcol;    // uniform format: the label of column j (RD_INF if the column is empty)
};

constexpr int kSpMaxAlpha = 16;        // lanes own alphas l+1 and l+9 of their 8-lane group
constexpr int kSpGroup = 8;            // lanes per output column

// Per-row finite spread of the output (for the next step's byte path): lanes keep packed
// running min (inf lanes are the largest value, so they never lower it) and max over finite
// values (inf lanes masked to 0); a CTA folds them per row pair and raises the flag if some
// row's max - min exceeds 254.
__device__ __forceinline__ void spread_update(uint32_t v, uint32_t &mn, uint32_t &mx) {
  mn = __vmins2(mn, v);
  mx = __vmaxs2(mx, v & ~__vcmpeq2(v, kInf2));
}

template <int NP>   // NP row pairs per CTA
__device__ __forceinline__ void spread_finish(uint32_t (&mn)[NP], uint32_t (&mx)[NP], int *flag,
                                              uint32_t (*smn)[NP], uint32_t (*smx)[NP]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < NP; ++r)
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mn[r] = __vmins2(mn[r], __shfl_xor_sync(0xffffffffu, mn[r], o));
      mx[r] = __vmaxs2(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], o));
    }
  if (lane == 0)
#pragma unroll
    for (int r = 0; r < NP; ++r) { smn[warp][r] = mn[r]; smx[warp][r] = mx[r]; }
  __syncthreads();
  if (threadIdx.x < NP) {
    const int r = threadIdx.x;
    uint32_t a = smn[0][r], b = smx[0][r];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { a = __vmins2(a, smn[w][r]); b = __vmaxs2(b, smx[w][r]); }
    const int lo0 = (int)(a & 0xFFFF), lo1 = (int)(a >> 16), hi0 = (int)(b & 0xFFFF), hi1 = (int)(b >> 16);
    if ((lo0 < RD_INF && hi0 - lo0 > 254) || (lo1 < RD_INF && hi1 - lo1 > 254)) atomicOr(flag, 1);
  }
}

// UNIFORM: every finite entry of column j carries the same label w_j (A(G): l(q,p) depends
// on p only), so the CSC holds bare shared-memory byte offsets, each column's list is
// padded to a multiple of 16 with the offset of an all-INF slot xs[Qc], two entries fold
// into one VIMNMX3 per row pair, and w_j is added once per column (min_q x_q + w = min_q
// (x_q + w)).  Otherwise (general labels, e.g. App. A) each entry carries its label.
template <bool STATS, int kSpThreads, int UNROLL, bool UNIFORM>
__global__ void __launch_bounds__(kSpThreads, 1)
minplus_sparse_kernel(const uint32_t *__restrict__ X, int64_t ld, SpArgs sa, uint32_t *__restrict__ C,
                      EpiArgs epi) {
  extern __shared__ __align__(16) uint2 xs[];
  __shared__ int32_t red[kSpThreads / 32][1 + 4 * kSpMaxAlpha];
  __shared__ uint32_t smn[kSpThreads / 32][2], smx[kSpThreads / 32][2];
  __shared__ int next_col;
  if (epi.spread_in && *epi.spread_in == 0) return;   // the byte kernel handles this step
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 3, sl = lane & 7;        // column group in the warp, lane in the group
  uint32_t smin2[2] = {kInf2, kInf2}, smax2[2] = {0, 0};
  const int64_t p0 = 2 * (int64_t)blockIdx.x;
  const uint32_t *x0 = X + p0 * ld, *x1 = x0 + ld;
  uint32_t *c0 = C + p0 * ld, *c1 = c0 + ld;
  const int64_t N = sa.N;
  constexpr int kWarps = kSpThreads / 32;
  const int64_t gi0 = epi.diag_row0 + 2 * p0;
  uint32_t lo2[2] = {0x7FFF7FFFu, 0x7FFF7FFFu}, hi2[2] = {0x80008000u, 0x80008000u}, mis[2] = {0, 0},
           fin[2] = {0, 0};
  int32_t dmin = INT_MAX;
  for (int ch = 0; ch < sa.nchunks; ++ch) {
    const int64_t q0 = (int64_t)ch * sa.Qc;
    const int qn = (int)min((int64_t)sa.Qc, N - q0);
    __syncthreads();
    for (int q = threadIdx.x; q < qn; q += kSpThreads) xs[q] = make_uint2(x0[q0 + q], x1[q0 + q]);
    if (UNIFORM && threadIdx.x == 0) xs[sa.Qc] = make_uint2(kInf2, kInf2);   // padding target
    __syncthreads();
    const int32_t *cp = sa.colptr + (int64_t)ch * (N + 1);
    const bool last = ch == sa.nchunks - 1;
    if (threadIdx.x == 0) next_col = 0;
    __syncthreads();
    // dynamic distribution: a warp grabs 4 consecutive columns (one per 8-lane group) at a
    // time, so warps stay balanced although column in-degrees vary by two orders
    for (;;) {
      int base = 0;
      if (lane == 0) base = atomicAdd(&next_col, 4);
      base = __shfl_sync(0xffffffffu, base, 0);
      if (base >= N) break;
      const int64_t j = base + g;
      const bool valid = j < N;
      int s = 0, e = 0;
      if (valid) { s = __ldg(cp + j); e = __ldg(cp + j + 1); }
      uint32_t a0 = kInf2, a1 = kInf2;
      if (valid && UNIFORM) {
        const uint32_t *ep = sa.ent + s + sl;
        const int cnt = e - s;                       // a multiple of 16
        const char *xb = reinterpret_cast<const char *>(xs);
#pragma unroll 2
        for (int t = 0; t < cnt; t += 2 * kSpGroup) {
          const uint32_t o0 = __ldg(ep + t), o1 = __ldg(ep + t + kSpGroup);
          const uint2 v0 = *reinterpret_cast<const uint2 *>(xb + o0);
          const uint2 v1 = *reinterpret_cast<const uint2 *>(xb + o1);
          a0 = __vimin3_s16x2(a0, v0.x, v1.x);
          a1 = __vimin3_s16x2(a1, v0.y, v1.y);
        }
      } else if (valid) {
        constexpr uint32_t kSent = (uint32_t)RD_INF << 17;   // q = 0, w = RD_INF: never wins
        for (int t = s + sl; t < e; t += UNROLL * kSpGroup) {
          uint32_t en[UNROLL];
#pragma unroll
          for (int u = 0; u < UNROLL; ++u)
            en[u] = (u == 0 || t + u * kSpGroup < e) ? __ldg(sa.ent + t + u * kSpGroup) : kSent;
#pragma unroll
          for (int u = 0; u < UNROLL; ++u) {
            const uint32_t w = en[u] >> 17;
            const uint2 xv = xs[en[u] & 0x1FFFFu];
            const uint32_t w2 = w | (w << 16);
            a0 = __viaddmin_s16x2(xv.x, w2, a0);
            a1 = __viaddmin_s16x2(xv.y, w2, a1);
          }
        }
      }
#pragma unroll
      for (int o = 4; o; o >>= 1) {
        a0 = __vmins2(a0, __shfl_xor_sync(0xffffffffu, a0, o));
        a1 = __vmins2(a1, __shfl_xor_sync(0xffffffffu, a1, o));
      }
      if (!valid) continue;
      if (ch > 0) {
        a0 = __vmins2(a0, c0[j]);
        a1 = __vmins2(a1, c1[j]);
      }
      if (UNIFORM && last) {   // + w_j, saturating at RD_INF: min(a + w, INF)
        const uint32_t w = (uint16_t)__ldg(sa.wcol + j);
        const uint32_t w2 = w | (w << 16);
        a0 = __viaddmin_s16x2(a0, w2, kInf2);
        a1 = __viaddmin_s16x2(a1, w2, kInf2);
      }
      if (sl == 0) c0[j] = a0;
      if (sl == 1) c1[j] = a1;
      if (last && sl == 0 && epi.spread_out) {
        spread_update(a0, smin2[0], smax2[0]);
        spread_update(a1, smin2[1], smax2[1]);
      }
      if (STATS && last) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int a = sl + 8 * h;
          if (a < epi.nprev) {
            const uint32_t *P = epi.prev[a];
            stats_pair(a0, P[p0 * ld + j], lo2[h], hi2[h], mis[h], fin[h]);
            stats_pair(a1, P[(p0 + 1) * ld + j], lo2[h], hi2[h], mis[h], fin[h]);
          }
        }
        if (sl == 0 && j >= gi0 && j < gi0 + 4) {
          const int t = (int)(j - gi0);
          const uint32_t w = t < 2 ? a0 : a1;
          dmin = min(dmin, (int)((w >> (16 * (t & 1))) & 0xFFFF));
        }
      }
    }
  }
  if (epi.spread_out) spread_finish<2>(smin2, smax2, epi.spread_out, smn, smx);
  if (!STATS) return;
  dmin = __reduce_min_sync(0xffffffffu, dmin);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    int32_t lo = min((int32_t)(int16_t)(lo2[h] & 0xFFFF), (int32_t)(int16_t)(lo2[h] >> 16));
    int32_t nhi = -max((int32_t)(int16_t)(hi2[h] & 0xFFFF), (int32_t)(int16_t)(hi2[h] >> 16));
    int32_t nm = mis[h] ? -1 : 0, nf = fin[h] ? -1 : 0;
    if (!fin[h]) { lo = INT_MAX; nhi = INT_MAX; }
    // combine the 4 column groups (lanes sl, sl+8, sl+16, sl+24 own the same alpha)
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      nhi = min(nhi, __shfl_xor_sync(0xffffffffu, nhi, o));
      nm = min(nm, __shfl_xor_sync(0xffffffffu, nm, o));
      nf = min(nf, __shfl_xor_sync(0xffffffffu, nf, o));
    }
    const int a = sl + 8 * h;
    if (g == 0 && a < epi.nprev) {
      red[warp][1 + 4 * a + 0] = lo;
      red[warp][1 + 4 * a + 1] = nhi;
      red[warp][1 + 4 * a + 2] = nm;
      red[warp][1 + 4 * a + 3] = nf;
    }
  }
  if (lane == 0) red[warp][0] = dmin;
  __syncthreads();
  for (int e = threadIdx.x; e < 1 + 4 * epi.nprev; e += kSpThreads) {
    int32_t v = red[0][e];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) v = min(v, red[w][e]);
    atomicMin(epi.stats + e, v);
  }
}

// The structured step with 8 rows per CTA stored as BYTES in shared memory (uniform labels
// only): byte r of xs[q] = X[row r][q] - base_r (the row's minimum over the q-chunk), 255 =
// inf; exact while every row's finite spread is <= 254 (flag spread_in == 0, computed by the
// previous step; V12: the spread is <= 16 from k = 4 on), otherwise the 16-bit kernel runs.
// Per gathered uint2 (8 rows) four PRMT expand the bytes into s16x2 pairs and two VIMNMX3 fold
// two entries; the group's minimum r gives base_r + r + w_j (255 -> inf).  Twice the rows of
// the 16-bit kernel for the same shared memory halves the per-column work per term.
template <bool STATS>
__global__ void __launch_bounds__(1024, 1)
minplus_sparse8_kernel(const uint32_t *__restrict__ X, int64_t ld, SpArgs sa, uint32_t *__restrict__ C,
                       EpiArgs epi) {
  constexpr int kT = 1024, kW = kT / 32;
  extern __shared__ __align__(16) uint2 xs[];
  __shared__ int32_t red[kW][1 + 4 * kSpMaxAlpha];
  __shared__ uint32_t smn[kW][4], smx[kW][4], sbase[4];
  __shared__ int next_col;
  if (*epi.spread_in != 0) return;                 // the 16-bit kernel handles this step
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 3, sl = lane & 7;
  const int64_t p0 = 4 * (int64_t)blockIdx.x;     // row pairs p0 .. p0+3 = rows 8b .. 8b+7
  const int64_t N = sa.N;
  const int64_t gi0 = epi.diag_row0 + 2 * p0;
  uint32_t lo2[2] = {0x7FFF7FFFu, 0x7FFF7FFFu}, hi2[2] = {0x80008000u, 0x80008000u}, mis[2] = {0, 0},
           fin[2] = {0, 0};
  uint32_t mn[4] = {kInf2, kInf2, kInf2, kInf2}, mx[4] = {0, 0, 0, 0};
  int32_t dmin = INT_MAX;
  const char *xb = reinterpret_cast<const char *>(xs);
  for (int ch = 0; ch < sa.nchunks; ++ch) {
    const int64_t q0 = (int64_t)ch * sa.Qc;
    const int qn = (int)min((int64_t)sa.Qc, N - q0);
    __syncthreads();
    // per-row minimum over the chunk (inf is the largest value)
    {
      uint32_t m4[4] = {kInf2, kInf2, kInf2, kInf2};
      for (int q = threadIdx.x; q < qn; q += kT)
#pragma unroll
        for (int r = 0; r < 4; ++r) m4[r] = __vmins2(m4[r], X[(p0 + r) * ld + q0 + q]);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int o = 16; o; o >>= 1) m4[r] = __vmins2(m4[r], __shfl_xor_sync(0xffffffffu, m4[r], o));
      if (lane == 0)
#pragma unroll
        for (int r = 0; r < 4; ++r) smn[warp][r] = m4[r];
      __syncthreads();
      if (threadIdx.x < 4) {
        uint32_t a = smn[0][threadIdx.x];
        for (int w = 1; w < kW; ++w) a = __vmins2(a, smn[w][threadIdx.x]);
        sbase[threadIdx.x] = a;
      }
      __syncthreads();
    }
    uint32_t base[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) base[r] = sbase[r];
    // bytes: x - base (finite, <= 254) or 255 (inf)
    for (int q = threadIdx.x; q < qn; q += kT) {
      uint32_t d[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint32_t x = X[(p0 + r) * ld + q0 + q];
        const uint32_t im = __vcmpeq2(x, kInf2);
        d[r] = (__vsub2(x, base[r]) & ~im) | (0x00FF00FFu & im);
      }
      xs[q] = make_uint2(__byte_perm(d[0], d[1], 0x6420), __byte_perm(d[2], d[3], 0x6420));
    }
    if (threadIdx.x == 0) xs[sa.Qc] = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);   // padding target
    if (threadIdx.x == 0) next_col = 0;
    __syncthreads();
    const int32_t *cp = sa.colptr + (int64_t)ch * (N + 1);
    const bool last = ch == sa.nchunks - 1;
    // software-pipelined column loop: the next batch is grabbed and its colptr loaded while the
    // current column's entries are walked; the label and the previous powers' entries for the
    // stats are requested before the walk so their latency overlaps it
    int bcol = 0;
    if (lane == 0) bcol = atomicAdd(&next_col, 4);
    bcol = __shfl_sync(0xffffffffu, bcol, 0);
    int s_n = 0, e_n = 0;
    if (bcol + g < N) { s_n = __ldg(cp + bcol + g); e_n = __ldg(cp + bcol + g + 1); }
    while (bcol < N) {
      const int64_t j = bcol + g;
      const bool valid = j < N;
      const int s = s_n, cnt = e_n - s_n;                             // cnt: a multiple of 16
      int nb = 0;
      if (lane == 0) nb = atomicAdd(&next_col, 4);
      nb = __shfl_sync(0xffffffffu, nb, 0);
      if (nb + g < N) { s_n = __ldg(cp + nb + g); e_n = __ldg(cp + nb + g + 1); }
      uint32_t wl = 0, pv[2][4];
      if (valid) {
        wl = (uint16_t)__ldg(sa.wcol + j);
        if (STATS && last) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int al = sl + 8 * h;
            const uint32_t *P = epi.prev[al < epi.nprev ? al : 0];
#pragma unroll
            for (int r = 0; r < 4; ++r) pv[h][r] = (al < epi.nprev) ? P[(p0 + r) * ld + j] : 0u;
          }
        }
      }
      bcol = nb;
      uint32_t a[4] = {0x00FF00FFu, 0x00FF00FFu, 0x00FF00FFu, 0x00FF00FFu};
      if (valid) {
        const uint32_t *ep = sa.ent + s + sl;
#pragma unroll 2
        for (int t = 0; t < cnt; t += 2 * kSpGroup) {
          const uint32_t o0 = __ldg(ep + t), o1 = __ldg(ep + t + kSpGroup);
          const uint2 v0 = *reinterpret_cast<const uint2 *>(xb + o0);
          const uint2 v1 = *reinterpret_cast<const uint2 *>(xb + o1);
          a[0] = __vimin3_s16x2(a[0], __byte_perm(v0.x, 0, 0x4140), __byte_perm(v1.x, 0, 0x4140));
          a[1] = __vimin3_s16x2(a[1], __byte_perm(v0.x, 0, 0x4342), __byte_perm(v1.x, 0, 0x4342));
          a[2] = __vimin3_s16x2(a[2], __byte_perm(v0.y, 0, 0x4140), __byte_perm(v1.y, 0, 0x4140));
          a[3] = __vimin3_s16x2(a[3], __byte_perm(v0.y, 0, 0x4342), __byte_perm(v1.y, 0, 0x4342));
        }
      }
#pragma unroll
      for (int o = 4; o; o >>= 1)
#pragma unroll
        for (int r = 0; r < 4; ++r) a[r] = __vmins2(a[r], __shfl_xor_sync(0xffffffffu, a[r], o));
      if (!valid) continue;
      const uint32_t w2 = wl | (wl << 16);
      uint32_t v[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {   // back to absolute: base + r + w (255 -> inf), saturating
        const uint32_t im = __vcmpeq2(a[r], 0x00FF00FFu);
        const uint32_t val = __vmins2(__vadd2(__vadd2(a[r], base[r]), w2), kInf2);
        v[r] = (val & ~im) | (kInf2 & im);
        if (ch > 0) v[r] = __vmins2(v[r], C[(p0 + r) * ld + j]);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (sl == r) C[(p0 + r) * ld + j] = v[r];
      if (last) {
        if (sl == 0)
#pragma unroll
          for (int r = 0; r < 4; ++r) spread_update(v[r], mn[r], mx[r]);
        if (STATS) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int al = sl + 8 * h;
            if (al < epi.nprev) {
#pragma unroll
              for (int r = 0; r < 4; ++r) stats_pair(v[r], pv[h][r], lo2[h], hi2[h], mis[h], fin[h]);
            }
          }
          if (sl == 0 && j >= gi0 && j < gi0 + 8) {
            const int t = (int)(j - gi0);
            dmin = min(dmin, (int)((v[t >> 1] >> (16 * (t & 1))) & 0xFFFF));
          }
        }
      }
    }
  }
  spread_finish<4>(mn, mx, epi.spread_out, smn, smx);
  if (!STATS) return;
  dmin = __reduce_min_sync(0xffffffffu, dmin);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    int32_t lo = min((int32_t)(int16_t)(lo2[h] & 0xFFFF), (int32_t)(int16_t)(lo2[h] >> 16));
    int32_t nhi = -max((int32_t)(int16_t)(hi2[h] & 0xFFFF), (int32_t)(int16_t)(hi2[h] >> 16));
    int32_t nm = mis[h] ? -1 : 0, nf = fin[h] ? -1 : 0;
    if (!fin[h]) { lo = INT_MAX; nhi = INT_MAX; }
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
      lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      nhi = min(nhi, __shfl_xor_sync(0xffffffffu, nhi, o));
      nm = min(nm, __shfl_xor_sync(0xffffffffu, nm, o));
      nf = min(nf, __shfl_xor_sync(0xffffffffu, nf, o));
    }
    const int al = sl + 8 * h;
    if (g == 0 && al < epi.nprev) {
      red[warp][1 + 4 * al + 0] = lo;
      red[warp][1 + 4 * al + 1] = nhi;
      red[warp][1 + 4 * al + 2] = nm;
      red[warp][1 + 4 * al + 3] = nf;
    }
  }
  if (lane == 0) red[warp][0] = dmin;
  __syncthreads();
  for (int e = threadIdx.x; e < 1 + 4 * epi.nprev; e += kT) {
    int32_t v = red[0][e];
    for (int w = 1; w < kW; ++w) v = min(v, red[w][e]);
    atomicMin(epi.stats + e, v);
  }
}

// The structured step in the slab layout (build_slab_layout): one LANE per output column
// (columns sorted by in-degree, so a warp's 32 lanes walk lists of nearly equal length), rows as
// bytes in shared memory as in minplus_sparse8_kernel.  Per 4 entries a lane issues 4 coalesced
// offset loads (one 128-byte line per warp each), 4 LDS.64 gathers, 16 PRMT and 8 VIMNMX3; a
// column has no cross-lane fold unless it was split (segmented shuffle min).  The step only
// produces C and the spread flag; diag and periodicity stats run after it (rp_diag_kernel,
// rp_stats_kernel), since here they would cost more than the product.
struct SlabArgs {
  const int4 *desc;        // per slab: entry offset, L (multiple of 4), head mask, 0
  const int32_t *lane_col; // per slab lane: output column j' or -1
  const uint32_t *ent8;    // lane-interleaved shared-memory slot pairs (rounds t, t+1)
  const int32_t *slab_start;
  int nchunks, Qc;
  int64_t N;
  const int16_t *wcol;
};

__global__ void __launch_bounds__(1024, 1)
minplus_slab8_kernel(const uint32_t *__restrict__ X, int64_t ld, SlabArgs sa, uint32_t *__restrict__ C,
                     const int *spread_in, int *spread_out) {
  constexpr int kT = 1024, kW = kT / 32;
  extern __shared__ __align__(16) uint2 xs[];
  __shared__ uint32_t smn[kW][4], smx[kW][4], sbase[4];
  __shared__ int next_slab;
  if (*spread_in != 0) return;                     // the 16-bit kernel handles this step
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p0 = 4 * (int64_t)blockIdx.x;     // row pairs p0 .. p0+3
  const int64_t N = sa.N;
  uint32_t mn[4] = {kInf2, kInf2, kInf2, kInf2}, mx[4] = {0, 0, 0, 0};
  for (int ch = 0; ch < sa.nchunks; ++ch) {
    const int64_t q0 = (int64_t)ch * sa.Qc;
    const int qn = (int)min((int64_t)sa.Qc, N - q0);
    __syncthreads();
    {
      uint32_t m4[4] = {kInf2, kInf2, kInf2, kInf2};
      for (int q = threadIdx.x; q < qn; q += kT)
#pragma unroll
        for (int r = 0; r < 4; ++r) m4[r] = __vmins2(m4[r], X[(p0 + r) * ld + q0 + q]);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int o = 16; o; o >>= 1) m4[r] = __vmins2(m4[r], __shfl_xor_sync(0xffffffffu, m4[r], o));
      if (lane == 0)
#pragma unroll
        for (int r = 0; r < 4; ++r) smn[warp][r] = m4[r];
      __syncthreads();
      if (threadIdx.x < 4) {
        uint32_t a = smn[0][threadIdx.x];
        for (int w = 1; w < kW; ++w) a = __vmins2(a, smn[w][threadIdx.x]);
        sbase[threadIdx.x] = a;
      }
      __syncthreads();
    }
    uint32_t base[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) base[r] = sbase[r];
    for (int q = threadIdx.x; q < qn; q += kT) {
      uint32_t d[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint32_t x = X[(p0 + r) * ld + q0 + q];
        const uint32_t im = __vcmpeq2(x, kInf2);
        d[r] = (__vsub2(x, base[r]) & ~im) | (0x00FF00FFu & im);
      }
      xs[q] = make_uint2(__byte_perm(d[0], d[1], 0x6420), __byte_perm(d[2], d[3], 0x6420));
    }
    if (threadIdx.x < 16) xs[sa.Qc + threadIdx.x] = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);   // sentinels
    if (threadIdx.x == 0) next_slab = 0;
    __syncthreads();
    const int s0 = sa.slab_start[ch], ns = sa.slab_start[ch + 1] - s0;
    const bool last = ch == sa.nchunks - 1;
    for (;;) {
      int s = 0;
      if (lane == 0) s = atomicAdd(&next_slab, 1);
      s = __shfl_sync(0xffffffffu, s, 0);
      if (s >= ns) break;
      const int4 d = __ldg(sa.desc + s0 + s);
      const int col = __ldg(sa.lane_col + (int64_t)(s0 + s) * 32 + lane);
      const uint32_t *ep = sa.ent8 + d.x + lane;
      // Fold without unpacking the bytes: as an unsigned 16-bit lane, (hi << 8 | lo) orders by
      // hi first, so the high byte of a lane-wise min is the min of the high bytes.  Raw words
      // give rows 1, 3 (5, 7) in the high bytes, words * 256 (IMAD, fma pipe) rows 0, 2 (4, 6).
      uint32_t ev0 = 0xFFFFFFFFu, od0 = 0xFFFFFFFFu, ev1 = 0xFFFFFFFFu, od1 = 0xFFFFFFFFu;
      for (int t = 0; t < d.y; t += 4) {
        const uint32_t w01 = __ldg(ep + (t / 2) * 32), w23 = __ldg(ep + (t / 2 + 1) * 32);
        const uint2 v0 = xs[w01 & 0xFFFFu], v1 = xs[w01 >> 16];
        const uint2 v2 = xs[w23 & 0xFFFFu], v3 = xs[w23 >> 16];
        od0 = __vimin3_u16x2(od0, v0.x, v1.x);
        od1 = __vimin3_u16x2(od1, v0.y, v1.y);
        ev0 = __vimin3_u16x2(ev0, v0.x * 256u, v1.x * 256u);
        ev1 = __vimin3_u16x2(ev1, v0.y * 256u, v1.y * 256u);
        od0 = __vimin3_u16x2(od0, v2.x, v3.x);
        od1 = __vimin3_u16x2(od1, v2.y, v3.y);
        ev0 = __vimin3_u16x2(ev0, v2.x * 256u, v3.x * 256u);
        ev1 = __vimin3_u16x2(ev1, v2.y * 256u, v3.y * 256u);
      }
      const uint32_t head = (uint32_t)d.z;
      if (head != 0xFFFFFFFFu) {   // split columns: segmented min towards each segment's head
        const uint32_t above = head & ~((2u << lane) - 1u);
        const int segend = above ? __ffs(above) - 1 : 32;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t u0 = __shfl_down_sync(0xffffffffu, ev0, o), u1 = __shfl_down_sync(0xffffffffu, od0, o);
          const uint32_t u2 = __shfl_down_sync(0xffffffffu, ev1, o), u3 = __shfl_down_sync(0xffffffffu, od1, o);
          if (lane + o < segend) {
            ev0 = __vminu2(ev0, u0); od0 = __vminu2(od0, u1);
            ev1 = __vminu2(ev1, u2); od1 = __vminu2(od1, u3);
          }
        }
      }
      if (col < 0 || !((head >> lane) & 1u)) continue;
      // high bytes -> row pairs (2r, 2r+1) as s16x2 byte offsets, 255 = inf
      uint32_t a[4];
      {
        const uint32_t e0 = (ev0 >> 8) & 0x00FF00FFu, q0 = (od0 >> 8) & 0x00FF00FFu;
        const uint32_t e1 = (ev1 >> 8) & 0x00FF00FFu, q1 = (od1 >> 8) & 0x00FF00FFu;
        a[0] = __byte_perm(e0, q0, 0x5410);
        a[1] = __byte_perm(e0, q0, 0x7632);
        a[2] = __byte_perm(e1, q1, 0x5410);
        a[3] = __byte_perm(e1, q1, 0x7632);
      }
      const uint32_t wl = (uint16_t)__ldg(sa.wcol + col);
      const uint32_t w2 = wl | (wl << 16);
#pragma unroll
      for (int r = 0; r < 4; ++r) {   // back to absolute: base + r + w (255 -> inf), saturating
        const uint32_t im = __vcmpeq2(a[r], 0x00FF00FFu);
        const uint32_t val = __vmins2(__vadd2(__vadd2(a[r], base[r]), w2), kInf2);
        uint32_t v = (val & ~im) | (kInf2 & im);
        uint32_t *cp = C + (p0 + r) * ld + col;
        if (ch > 0) v = __vmins2(v, *cp);
        *cp = v;
        if (last) spread_update(v, mn[r], mx[r]);
      }
    }
  }
  spread_finish<4>(mn, mx, spread_out, smn, smx);
}

// diag[k] for a row panel in RP layout whose columns are permuted (inv: state -> column;
// nullptr = identity): min over local rows i of X[i][inv[r0 + i]].
__global__ void rp_diag_kernel(const uint32_t *__restrict__ X, int64_t ld, int64_t rows, int64_t r0,
                               const int32_t *__restrict__ inv, int32_t *stats) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int32_t v = INT_MAX;
  if (i < rows) {
    const int64_t j = inv ? inv[r0 + i] : r0 + i;
    const uint32_t w = X[(i >> 1) * ld + j];
    v = (int32_t)((i & 1) ? (w >> 16) : (w & 0xFFFF));
  }
  v = __reduce_min_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && v != INT_MAX) atomicMin(stats, v);
}

// Periodicity stats of an RP panel against earlier powers (rd_chain_step layout, entries
// 1..4*nprev; elementwise, so any consistent layout works).  Warp w of a block owns alpha w+1,
// lanes take 16-byte column chunks, a block sweeps (row pair, 128-column block) items and the
// current power's line is re-served from L1 to the 16 warps.
//   SAMPLE: only row pairs with (p / 4) % stride == 0 (a fixed subset of rows).
//   otherwise: every row pair, but only alphas the vector does not already prove aperiodic
//   (a subset that is not uniform proves the whole is not; a "survivor" is recomputed in full
//   and MIN-merged — min over subset and full = full).  Blocks that see a survivor turn into a
//   non-survivor while others merge skip it: it is proven aperiodic by then.
template <bool SAMPLE>
__global__ void __launch_bounds__(512) rp_stats_kernel(const uint32_t *__restrict__ cur, int64_t ld,
                                                       int64_t pairs, int64_t cols, int stride,
                                                       PanelStatsArgs pa, int32_t *stats) {
  __shared__ int any;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bool mine = warp < pa.nprev;
  if (!SAMPLE) {
    if (mine) {
      const volatile int32_t *s = stats + 1 + 4 * warp;
      const int32_t lo = s[0], nhi = s[1], nmis = s[2], nfin = s[3];
      mine = nmis == 0 && (nfin == 0 || lo == -nhi);
    }
    if (threadIdx.x == 0) any = 0;
    __syncthreads();
    if (mine && lane == 0) any = 1;
    __syncthreads();
    if (!any) return;
  }
  if (!mine) return;     // no barrier below: warps without an alpha to test leave at once
  const uint32_t *P = reinterpret_cast<const uint32_t *>(pa.prev[warp]);
  uint32_t lo2 = 0x7FFF7FFFu, hi2 = 0x80008000u, mis = 0, fin = 0;
  const int64_t nb = (cols + 127) / 128;
  const int64_t np = SAMPLE ? ((pairs + 4LL * stride - 1) / (4LL * stride)) * 4 : pairs;
  const int64_t items = np * nb;
  for (int64_t v = blockIdx.x; v < items; v += gridDim.x) {
    const int64_t ip = v / nb;
    const int64_t p = SAMPLE ? (ip / 4) * 4 * stride + (ip & 3) : ip;
    const int64_t j = (v - ip * nb) * 128 + lane * 4;
    if (p >= pairs || j >= cols) continue;
    const uint4 x = *reinterpret_cast<const uint4 *>(cur + p * ld + j);
    const uint4 y = *reinterpret_cast<const uint4 *>(P + p * ld + j);
    stats_pair(x.x, y.x, lo2, hi2, mis, fin);
    stats_pair(x.y, y.y, lo2, hi2, mis, fin);
    stats_pair(x.z, y.z, lo2, hi2, mis, fin);
    stats_pair(x.w, y.w, lo2, hi2, mis, fin);
  }
  int32_t lo = min((int32_t)(int16_t)(lo2 & 0xFFFF), (int32_t)(int16_t)(lo2 >> 16));
  int32_t hi = max((int32_t)(int16_t)(hi2 & 0xFFFF), (int32_t)(int16_t)(hi2 >> 16));
  if (!fin) { lo = INT_MAX; hi = INT_MIN + 1; }
  const int32_t v0 = __reduce_min_sync(0xffffffffu, lo);
  const int32_t v1 = __reduce_min_sync(0xffffffffu, -hi);
  const int32_t v2 = __reduce_min_sync(0xffffffffu, mis ? -1 : 0);
  const int32_t v3 = __reduce_min_sync(0xffffffffu, fin ? -1 : 0);
  if (lane == 0) {
    atomicMin(stats + 1 + 4 * warp, v0);
    atomicMin(stats + 2 + 4 * warp, v1);
    atomicMin(stats + 3 + 4 * warp, v2);
    atomicMin(stats + 4 + 4 * warp, v3);
  }
}

// Row-major int16 rows [row0, row0+rows) of X (ld) -> RP u32 [pairs][ldr], INF padded.
__global__ void pack_rp_kernel(const int16_t *__restrict__ X, int64_t ld, int64_t rows, int64_t cols,
                               int64_t row0, uint32_t *__restrict__ RP, int64_t ldr, int64_t pairs) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, p = blockIdx.y;
  if (j >= ldr || p >= pairs) return;
  uint32_t lo = RD_INF, hi = RD_INF;
  if (j < cols) {
    if (2 * p < rows) lo = (uint32_t)min((int)X[(row0 + 2 * p) * ld + j], (int)RD_INF);
    if (2 * p + 1 < rows) hi = (uint32_t)min((int)X[(row0 + 2 * p + 1) * ld + j], (int)RD_INF);
  }
  RP[p * ldr + j] = lo | (hi << 16);
}

// Dense-chain operands straight from a general-format CSC of A (per q-chunk: entries hold
// q - ch * Qc in 17 bits, so orders with N >= 2^17 take several chunks), thread per column,
// into all-INF buffers: the packed right operand BP[t][j] = A[2t][j] | A[2t+1][j] << 16 and the
// PM panel XT[t][i] = A[r0+i][2t] | A[r0+i][2t+1] << 16 of rows [r0, r1).
__global__ void scatter_dense_operands_kernel(const int32_t *__restrict__ colptr, const uint32_t *__restrict__ ent,
                                              int64_t N, int nchunks, int Qc, uint32_t *__restrict__ BP,
                                              int64_t ldp, uint32_t *__restrict__ XT, int64_t ldt, int64_t r0,
                                              int64_t r1) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  uint16_t *hb = reinterpret_cast<uint16_t *>(BP), *hx = reinterpret_cast<uint16_t *>(XT);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int32_t *cp = colptr + (int64_t)ch * (N + 1);
    for (int t = cp[j]; t < cp[j + 1]; ++t) {
      const int64_t q = (int64_t)ch * Qc + (ent[t] & 0x1FFFFu);
      const uint16_t w = (uint16_t)(ent[t] >> 17);
      if (BP) hb[((q >> 1) * ldp + j) * 2 + (q & 1)] = w;
      if (XT && q >= r0 && q < r1) hx[((j >> 1) * ldt + (q - r0)) * 2 + (j & 1)] = w;
    }
  }
}

// q-chunking of a general-format CSC: entries store q - ch * Qc in 17 bits
inline void csc_chunks_17bit(int64_t N, int *nchunks, int *Qc) {
  *nchunks = (int)((N + (1 << 17) - 1) >> 17);
  *Qc = (int)((N + *nchunks - 1) / *nchunks);
}

// A^1 rows [r0, r1) into an all-INF RP slot straight from the CSC (thread per column).
__global__ void scatter_rp_kernel(const int32_t *__restrict__ colptr, const uint32_t *__restrict__ ent, int64_t N,
                                  int nchunks, int Qc, int64_t r0, int64_t r1, uint32_t *__restrict__ RP,
                                  int64_t ldr, const int16_t *__restrict__ wcol,
                                  const int32_t *__restrict__ perm) {   // perm: CSC row q' -> state
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  uint16_t *h = reinterpret_cast<uint16_t *>(RP);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int32_t *cp = colptr + (int64_t)ch * (N + 1);
    for (int t = cp[j]; t < cp[j + 1]; ++t) {
      int64_t ql;
      uint16_t w;
      if (wcol) {                                   // uniform: byte offsets, padding = Qc * 8
        ql = ent[t] >> 3;
        if (ql >= Qc) continue;
        w = (uint16_t)wcol[j];
      } else {
        ql = ent[t] & 0x1FFFFu;
        w = (uint16_t)(ent[t] >> 17);
      }
      int64_t q = (int64_t)ch * Qc + ql;
      if (perm) q = perm[q];
      if (q < r0 || q >= r1) continue;
      const int64_t i = q - r0;
      h[((i >> 1) * ldr + j) * 2 + (i & 1)] = w;
    }
  }
}

// RP -> row-major int16 rows x cols (inv: state -> stored column, nullptr = identity)
__global__ void unpack_rp_kernel(const uint32_t *__restrict__ RP, int64_t ldr, int64_t rows, int64_t cols,
                                 int16_t *__restrict__ X, const int32_t *__restrict__ inv) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
  if (i >= rows || j >= cols) return;
  const uint32_t w = RP[(i >> 1) * ldr + (inv ? inv[j] : j)];
  X[i * cols + j] = (int16_t)((i & 1) ? (w >> 16) : (w & 0xFFFF));
}

}  // namespace

namespace {
constexpr int kSpSmemMax = 216 * 1024;  // dynamic smem for xs (static red[] + counter aside: <= 8.2 KB)

// CSC of the right operand per q-chunk, from the row-major host matrix (OpenMP over
// column blocks).  Entries (q - q0) | w << 17, q ascending within a column.
void build_csc(const int16_t *A, int64_t N, int nchunks, int Qc, std::vector<int32_t> &colptr,
               std::vector<uint32_t> &ent) {
  colptr.assign((size_t)nchunks * (N + 1), 0);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int64_t q0 = (int64_t)ch * Qc, q1 = std::min(N, q0 + Qc);
    int32_t *cp = colptr.data() + (size_t)ch * (N + 1);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t jb = 0; jb < N; jb += 256) {
      const int64_t je = std::min(N, jb + 256);
      for (int64_t q = q0; q < q1; ++q) {
        const int16_t *row = A + q * N;
        for (int64_t j = jb; j < je; ++j)
          if (row[j] < RD_INF) cp[j + 1]++;
      }
    }
  }
  int64_t total = 0;
  for (int ch = 0; ch < nchunks; ++ch) {
    int32_t *cp = colptr.data() + (size_t)ch * (N + 1);
    cp[0] = (int32_t)total;
    for (int64_t j = 0; j < N; ++j) { total += cp[j + 1]; cp[j + 1] = (int32_t)total; }
  }
  ent.assign((size_t)std::max<int64_t>(total, 1), 0);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int64_t q0 = (int64_t)ch * Qc, q1 = std::min(N, q0 + Qc);
    const int32_t *cp = colptr.data() + (size_t)ch * (N + 1);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t jb = 0; jb < N; jb += 256) {
      const int64_t je = std::min(N, jb + 256);
      std::vector<int32_t> pos(cp + jb, cp + je);
      for (int64_t q = q0; q < q1; ++q) {
        const int16_t *row = A + q * N;
        for (int64_t j = jb; j < je; ++j)
          if (row[j] < RD_INF) ent[pos[j - jb]++] = (uint32_t)(q - q0) | ((uint32_t)row[j] << 17);
      }
    }
  }
}
// Re-encodes a general CSC (entries (q - q0) | w << 17) in the uniform-label format if every
// column's entries share one label: entries (q - q0) * 8 (shared-memory byte offsets), each
// column's list per chunk padded to a multiple of 16 with Qc * 8, wcol[j] = the label
// (RD_INF for an empty column).  Returns false (inputs untouched) if some column mixes labels.
bool csc_to_uniform(int64_t N, int nchunks, int Qc, std::vector<int32_t> &colptr, std::vector<uint32_t> &ent,
                    std::vector<int16_t> &wcol) {
  std::vector<int32_t> w((size_t)N, -1);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int32_t *cp = colptr.data() + (size_t)ch * (N + 1);
    for (int64_t j = 0; j < N; ++j)
      for (int32_t t = cp[j]; t < cp[j + 1]; ++t) {
        const int32_t lab = (int32_t)(ent[t] >> 17);
        if (w[j] < 0) w[j] = lab;
        else if (w[j] != lab) return false;
      }
  }
  std::vector<int32_t> ucp((size_t)nchunks * (N + 1), 0);
  int64_t total = 0;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int32_t *cp = colptr.data() + (size_t)ch * (N + 1);
    int32_t *up = ucp.data() + (size_t)ch * (N + 1);
    up[0] = (int32_t)total;
    for (int64_t j = 0; j < N; ++j) {
      total += (cp[j + 1] - cp[j] + 15) / 16 * 16;
      up[j + 1] = (int32_t)total;
    }
  }
  std::vector<uint32_t> uent((size_t)std::max<int64_t>(total, 1), (uint32_t)Qc * 8u);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int32_t *cp = colptr.data() + (size_t)ch * (N + 1);
    const int32_t *up = ucp.data() + (size_t)ch * (N + 1);
    for (int64_t j = 0; j < N; ++j)
      for (int32_t t = cp[j]; t < cp[j + 1]; ++t) uent[up[j] + (t - cp[j])] = (ent[t] & 0x1FFFFu) * 8u;
  }
  wcol.assign((size_t)N, RD_INF);
  for (int64_t j = 0; j < N; ++j)
    if (w[j] >= 0) wcol[j] = (int16_t)w[j];
  colptr.swap(ucp);
  ent.swap(uent);
  return true;
}

// Slab layout of the structured step (minplus_slab8_kernel).  The chain runs in a column-
// permuted basis: X'_k = A^k P^T with P sorting the states by in-degree (descending), so that
// C' = X' (x) A' with A' = P A P^T (rows of the powers stay in natural order; diag and the
// periodicity test are invariant).  Per q'-chunk the columns j' are dealt to
// warp lanes in order, 32 per slab; a column longer than T is split over adjacent lanes of one
// slab (segments, folded by a segmented shuffle min).  Entries are stored lane-interleaved,
// ent8[off + (t/2)*32 + lane] = the slots ql of that lane's entries in rounds t and t+1 as two
// u16 (Qc .. Qc+15 = inf padding), so a warp reads one coalesced 128-byte line per two rounds.
struct SlabHost {
  std::vector<int32_t> perm, inv;         // new column -> state, state -> new column
  std::vector<int32_t> ucolptr;           // uniform CSC in the new basis (16-bit fallback kernel)
  std::vector<uint32_t> uent;
  std::vector<int16_t> wcol;              // label of new column j'
  std::vector<int32_t> desc;              // per slab: off, L, headmask, 0
  std::vector<int32_t> lane_col;          // per slab lane: j' or -1
  std::vector<uint32_t> ent8;
  std::vector<int32_t> slab_start;        // per chunk, nchunks + 1
};

// One slab of the slab layout: the lanes' pieces (column, first index into lists, length),
// scheduled into L rounds (multiple of 4) of bank-conflict-free gathers; out = L x 32 byte
// offsets (lane-interleaved).  Returns false if some entry was not scheduled exactly once.
struct SlabPiece { int32_t col; int64_t b; int32_t len; bool head; };
static bool colour_slab(const std::vector<SlabPiece> &cur, const int32_t *lists, int Qc,
                        std::vector<uint32_t> &out, int32_t &Lout) {
  bool colour_ok = true;
  // per half-warp, schedule the entries into rounds so that no two lanes of the half-warp
  // read different slots of one bank pair in a round (8-byte slot q uses banks 2q, 2q+1:
  // class q mod 16): a proper edge colouring of the bipartite multigraph lanes x classes
  // with Delta colours (Koenig's theorem; alternating-path recolouring)
  std::vector<std::vector<int32_t>> rounds(32);   // rounds[lane][r] = slot or -1
  int32_t L = 0;
  for (int h = 0; h < 2; ++h) {
    int D = 0;
    int dv[16] = {0};
    for (int u = 0; u < 16; ++u) {
      const int l = 16 * h + u;
      if (l >= (int)cur.size()) continue;
      D = std::max(D, (int)cur[l].len);
      for (int32_t t = 0; t < cur[l].len; ++t) D = std::max(D, ++dv[lists[cur[l].b + t] & 15]);
    }
    std::vector<int32_t> cu((size_t)16 * D, -1), cq((size_t)16 * D, -1), cv((size_t)16 * D, -1);
    auto freeU = [&](int u) { int c = 0; while (cu[(size_t)u * D + c] >= 0) ++c; return c; };
    auto freeV = [&](int v) { int c = 0; while (cv[(size_t)v * D + c] >= 0) ++c; return c; };
    struct E { int u, v, c; int32_t q; };
    std::vector<E> path;
    for (int u = 0; u < 16; ++u) {
      const int l = 16 * h + u;
      if (l >= (int)cur.size()) continue;
      for (int32_t t = 0; t < cur[l].len; ++t) {
        const int32_t q = lists[cur[l].b + t];
        const int v = q & 15;
        const int a = freeU(u), b = freeV(v);
        if (cv[(size_t)v * D + a] >= 0) {
          // swap colours a <-> b along the alternating path from v (a, b, a, ...); it
          // cannot reach u (bipartite parity), so a becomes free at both ends
          path.clear();
          int x = v, c = a;
          bool onV = true;
          for (;;) {
            if (onV) {
              const int y = cv[(size_t)x * D + c];
              if (y < 0) break;
              path.push_back(E{y, x, c, cq[(size_t)y * D + c]});
              x = y;
            } else {
              const int y = cu[(size_t)x * D + c];
              if (y < 0) break;
              path.push_back(E{x, y, c, cq[(size_t)x * D + c]});
              x = y;
            }
            onV = !onV;
            c = (c == a) ? b : a;
          }
          for (auto &e : path) {
            cu[(size_t)e.u * D + e.c] = -1;
            cq[(size_t)e.u * D + e.c] = -1;
            cv[(size_t)e.v * D + e.c] = -1;
          }
          for (auto &e : path) {
            const int nc = e.c == a ? b : a;
            cu[(size_t)e.u * D + nc] = e.v;
            cq[(size_t)e.u * D + nc] = e.q;
            cv[(size_t)e.v * D + nc] = e.u;
          }
        }
        cu[(size_t)u * D + a] = v;
        cq[(size_t)u * D + a] = q;
        cv[(size_t)v * D + a] = u;
      }
    }
    for (int u = 0; u < 16; ++u) {
      const int l = 16 * h + u;
      rounds[l].assign((size_t)D, -1);
      if (l >= (int)cur.size()) continue;
      int32_t got = 0;
      for (int c = 0; c < D; ++c) got += (rounds[l][c] = cq[(size_t)u * D + c]) >= 0;
      if (got != cur[l].len) colour_ok = false;   // every entry scheduled exactly once
    }
    L = std::max(L, (int32_t)D);
  }
  L = (L + 3) / 4 * 4;
  const uint32_t pad = (uint32_t)Qc * 8u;
  out.assign((size_t)L * 32, pad);
  for (int h = 0; h < 2; ++h)
    for (int32_t r = 0; r < L; ++r) {
      bool used[16] = {false};
      for (int u = 0; u < 16; ++u) {
        const auto &R = rounds[16 * h + u];
        if (r < (int32_t)R.size() && R[r] >= 0) used[R[r] & 15] = true;
      }
      int fc = 0;
      while (fc < 15 && used[fc]) ++fc;
      // padding reads the inf sentinel (slots Qc .. Qc+15, one per class) of a class no real
      // entry of the half-warp uses in this round
      const uint32_t sent = (uint32_t)(Qc + ((fc - Qc % 16 + 32) % 16)) * 8u;
      for (int u = 0; u < 16; ++u) {
        const int l = 16 * h + u;
        const auto &R = rounds[l];
        const bool real = r < (int32_t)R.size() && R[r] >= 0;
        out[(size_t)r * 32 + l] = real ? (uint32_t)R[r] * 8u : sent;
      }
    }
  Lout = L;
  return colour_ok;
}

// From the natural general-format CSC (entries (q - q0) | w << 17, chunks of Qc).  Returns
// false if some column mixes labels (then the chain keeps the natural basis).
bool build_slab_layout(int64_t N, int nchunks, int Qc, const std::vector<int32_t> &colptr,
                       const std::vector<uint32_t> &ent, SlabHost &S) {
  std::vector<int32_t> deg((size_t)N, 0), lab((size_t)N, -1);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int32_t *cp = colptr.data() + (size_t)ch * (N + 1);
    for (int64_t j = 0; j < N; ++j) {
      deg[j] += cp[j + 1] - cp[j];
      for (int32_t t = cp[j]; t < cp[j + 1]; ++t) {
        const int32_t w = (int32_t)(ent[t] >> 17);
        if (lab[j] < 0) lab[j] = w;
        else if (lab[j] != w) return false;
      }
    }
  }
  S.perm.resize((size_t)N);
  for (int64_t j = 0; j < N; ++j) S.perm[j] = (int32_t)j;
  std::stable_sort(S.perm.begin(), S.perm.end(), [&](int32_t a, int32_t b) { return deg[a] > deg[b]; });
  S.inv.resize((size_t)N);
  for (int64_t j = 0; j < N; ++j) S.inv[S.perm[j]] = (int32_t)j;
  S.wcol.assign((size_t)N, RD_INF);
  for (int64_t j = 0; j < N; ++j)
    if (lab[S.perm[j]] >= 0) S.wcol[j] = (int16_t)lab[S.perm[j]];
  // lists per (new chunk, new column) of ql = q' - chunk start, ascending
  std::vector<int32_t> cnt((size_t)nchunks * N, 0);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int32_t *cp = colptr.data() + (size_t)ch * (N + 1);
    for (int64_t j = 0; j < N; ++j)
      for (int32_t t = cp[j]; t < cp[j + 1]; ++t) {
        const int64_t q = (int64_t)ch * Qc + (ent[t] & 0x1FFFFu), qn = S.inv[q];
        cnt[(size_t)(qn / Qc) * N + S.inv[j]]++;
      }
  }
  std::vector<int64_t> lp((size_t)nchunks * N + 1, 0);
  for (size_t i = 0; i < cnt.size(); ++i) lp[i + 1] = lp[i] + cnt[i];
  std::vector<int32_t> lists((size_t)std::max<int64_t>(lp.back(), 1));
  {
    std::vector<int64_t> pos(lp.begin(), lp.end() - 1);
    for (int ch = 0; ch < nchunks; ++ch) {
      const int32_t *cp = colptr.data() + (size_t)ch * (N + 1);
      for (int64_t j = 0; j < N; ++j)
        for (int32_t t = cp[j]; t < cp[j + 1]; ++t) {
          const int64_t q = (int64_t)ch * Qc + (ent[t] & 0x1FFFFu), qn = S.inv[q];
          const int64_t c = qn / Qc;
          lists[pos[(size_t)c * N + S.inv[j]]++] = (int32_t)(qn - c * Qc);
        }
    }
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < (int64_t)cnt.size(); ++i) std::sort(lists.begin() + lp[i], lists.begin() + lp[i + 1]);
  }
  const uint32_t pad = (uint32_t)Qc * 8u;
  // uniform CSC (lists padded to 16) for the 16-bit fallback kernel
  S.ucolptr.assign((size_t)nchunks * (N + 1), 0);
  int64_t total = 0;
  for (int ch = 0; ch < nchunks; ++ch) {
    int32_t *up = S.ucolptr.data() + (size_t)ch * (N + 1);
    up[0] = (int32_t)total;
    for (int64_t j = 0; j < N; ++j) {
      total += (cnt[(size_t)ch * N + j] + 15) / 16 * 16;
      up[j + 1] = (int32_t)total;
    }
  }
  S.uent.assign((size_t)std::max<int64_t>(total, 1), pad);
  for (int ch = 0; ch < nchunks; ++ch)
    for (int64_t j = 0; j < N; ++j) {
      const size_t li = (size_t)ch * N + j;
      const int32_t u0 = S.ucolptr[(size_t)ch * (N + 1) + j];
      for (int64_t t = lp[li]; t < lp[li + 1]; ++t) S.uent[u0 + (t - lp[li])] = (uint32_t)lists[t] * 8u;
    }
  // slabs: columns dealt to lanes in order (sequential), each slab scheduled in parallel
  S.desc.clear(); S.lane_col.clear(); S.ent8.clear();
  S.slab_start.assign((size_t)nchunks + 1, 0);
  std::vector<std::vector<SlabPiece>> slabs;
  for (int ch = 0; ch < nchunks; ++ch) {
    S.slab_start[ch] = (int32_t)slabs.size();
    int64_t maxlen = 0;
    for (int64_t j = 0; j < N; ++j) maxlen = std::max<int64_t>(maxlen, cnt[(size_t)ch * N + j]);
    const int64_t T = std::max<int64_t>(256, (maxlen + 31) / 32);
    std::vector<SlabPiece> cur;
    for (int64_t j = 0; j < N; ++j) {
      const size_t li = (size_t)ch * N + j;
      const int64_t d = cnt[li];
      const int64_t pieces = d <= T ? 1 : (d + T - 1) / T;
      if ((int64_t)cur.size() + pieces > 32) { slabs.push_back(std::move(cur)); cur.clear(); }
      const int64_t per = pieces == 1 ? d : (d + pieces - 1) / pieces;
      for (int64_t p = 0; p < pieces; ++p) {
        const int64_t b = p * per, e = std::min<int64_t>(d, b + per);
        cur.push_back(SlabPiece{(int32_t)j, lp[li] + b, (int32_t)std::max<int64_t>(0, e - b), p == 0});
      }
      if (cur.size() == 32) { slabs.push_back(std::move(cur)); cur.clear(); }
    }
    if (!cur.empty()) slabs.push_back(std::move(cur));
  }
  const int64_t ns = (int64_t)slabs.size();
  std::vector<std::vector<uint32_t>> sent8((size_t)ns);
  std::vector<int32_t> sL((size_t)ns, 0);
  bool all_ok = true;
#pragma omp parallel for schedule(dynamic, 16) reduction(&& : all_ok)
  for (int64_t s = 0; s < ns; ++s) all_ok = colour_slab(slabs[s], lists.data(), Qc, sent8[s], sL[s]) && all_ok;
  if (!all_ok) return false;
  // two rounds per word: slot indices (byte offset / 8, < Qc + 16 <= 27664) of rounds t, t+1
  int64_t total2 = 0;
  for (int64_t s = 0; s < ns; ++s) total2 += (int64_t)sL[s] * 16;
  S.ent8.resize((size_t)std::max<int64_t>(total2, 1), (pad / 8) * 0x10001u);
  S.desc.resize((size_t)ns * 4);
  S.lane_col.resize((size_t)ns * 32);
  int64_t off = 0;
  for (int64_t s = 0; s < ns; ++s) {
    for (int32_t r = 0; r < sL[s]; r += 2)
      for (int l = 0; l < 32; ++l)
        S.ent8[off + (int64_t)(r / 2) * 32 + l] =
            (sent8[s][(size_t)r * 32 + l] >> 3) | ((sent8[s][(size_t)(r + 1) * 32 + l] >> 3) << 16);
    uint32_t head = 0;
    for (int l = 0; l < 32; ++l) {
      const bool real = l < (int)slabs[s].size();
      if (!real || slabs[s][l].head) head |= 1u << l;
      S.lane_col[(size_t)s * 32 + l] = real ? slabs[s][l].col : -1;
    }
    S.desc[(size_t)s * 4 + 0] = (int32_t)off;
    S.desc[(size_t)s * 4 + 1] = sL[s];
    S.desc[(size_t)s * 4 + 2] = (int32_t)head;
    S.desc[(size_t)s * 4 + 3] = 0;
    off += (int64_t)sL[s] * 16;
  }
  S.slab_start[nchunks] = (int32_t)ns;
  return true;
}
}  // namespace

// Host slab layout of A(G) for words of length m, built from the successor generator once per
// process and shared by later chains of the same order (e.g. the row panels of
// dist.power_sequence_panels: 4 panels at m = 11 rebuilt it for 7 s each).  One entry.
struct SlabCached {
  int m = 0, nchunks = 0, Qc = 0;
  bool border = false;
  int64_t nnz = 0;
  std::vector<int16_t> dg;
  SlabHost S;
};
static std::mutex g_slab_mu;
static std::shared_ptr<const SlabCached> g_slab_cache;

static std::shared_ptr<const SlabCached> slab_cached(int m, bool border, int nchunks, int Qc) {
  std::lock_guard<std::mutex> lk(g_slab_mu);
  const auto &g = g_slab_cache;
  if (g && g->m == m && g->border == border && g->nchunks == nchunks && g->Qc == Qc) return g;
  g_slab_cache.reset();                                  // release the old layout first
  auto n = std::make_shared<SlabCached>();
  n->m = m; n->border = border; n->nchunks = nchunks; n->Qc = Qc;
  std::vector<int32_t> colptr;
  std::vector<uint32_t> ent;
  build_csc_direct(m, border, nchunks, Qc, colptr, ent, n->dg);
  n->nnz = colptr.back();
  const int64_t N = (int64_t)n->dg.size();
  if (!build_slab_layout(N, nchunks, Qc, colptr, ent, n->S)) return nullptr;
  g_slab_cache = n;
  return n;
}

// ================================================================ power chain ==
struct rd_chain {
  int m = 0, alpha_max = 0, k = 0, device = 0, method = 0;
  int64_t N = 0, P = 0, r0 = 0, r1 = 0, Mr = 0, Mp = 0;
  cudaStream_t st = nullptr;
  uint32_t *BP = nullptr;    // method 0: packed A, [P/2][P]
  uint32_t *ring = nullptr;  // method 0: (alpha_max+1) PM slots [P/2][Mp]; method 1: RP slots [Mp/2][P]
  int64_t slot_words = 0;
  int32_t diag1 = INT32_MAX;  // min_p A_pp (self-loop labels), for diag[1]
  // method 1 (structured step): CSC of A per q-chunk
  int32_t *colptr = nullptr;
  uint32_t *ent = nullptr;
  int16_t *wcol = nullptr;   // uniform-label format (see minplus_sparse_kernel)
  uint32_t *ws = nullptr;    // method 0 split-K partial tiles (small grids), lazily allocated
  int *tile_cnt = nullptr;   // method 0 split-K fixup tickets, one per tile (self-resetting)
  // method 0, long steps: the DPX column count is tuned on the chain's first two TMA steps
  // (3, then 4, each timed with events; the faster is kept) unless rd_set_gemm_variant fixed it
  int dpx = -1, tune_state = 0;
  cudaEvent_t tune_ev[16] = {};
  int nsplit = 1;
  int *spread = nullptr;     // method 1 byte path: flags[k & 1] = "some row of A^k spreads > 254"
  // method 1 slab layout (build_slab_layout): columns of the powers permuted, inv = state ->
  // column; the 16-bit fallback reads colptr/ent/wcol in the same basis
  int32_t *perm = nullptr, *inv = nullptr, *lane_col = nullptr, *slab_start = nullptr;
  int4 *desc = nullptr;
  uint32_t *ent8 = nullptr;
  int nchunks = 0, Qc = 0;
  int64_t nnz = 0;
  std::vector<void *> pooled;   // buffers taken from the library's stream-ordered pool
  TmaOps tma{};                 // dense chains: tensor maps of the ring and packed operand
  bool tma_ready = false;
  uint32_t *slot(int k) const { return ring + (int64_t)(k % (alpha_max + 1)) * slot_words; }
};

// Device memory of chains.  cudaMalloc / cudaFree cost 0.05-20 ms each for small buffers
// and up to ~1 s to unmap a 10 GB ring, depending on the driver's state, while a small-order
// chain computes in ~0.5 ms (m = 5).  Chain buffers come from a library-owned stream-ordered
// pool instead (µs once warm); up to kPoolKeep bytes stay mapped between chains (an m = 9
// dense chain's ring + packed operand is 11.7 GB), anything beyond is returned at the next
// synchronisation.  Buffers above kPoolMax (the m >= 10 rings: growing the pool by 92 GB took
// 9 s against 0.5 s for cudaMalloc) and allocations the pool cannot serve use cudaMalloc.
template <typename T>
static cudaError_t chain_malloc(rd_chain *c, T **p, size_t bytes) {
  *p = nullptr;
  if (bytes <= kPoolMax) {
    if (cudaMemPool_t pool = chain_pool(c->device)) {
      void *q = nullptr;
      if (cudaMallocFromPoolAsync(&q, bytes, pool, c->st) == cudaSuccess) {
        c->pooled.push_back(q);
        *p = reinterpret_cast<T *>(q);
        return cudaSuccess;
      }
      (void)cudaGetLastError();
    }
  }
  void *q = nullptr;
  cudaError_t e = cudaMalloc(&q, bytes);
  *p = reinterpret_cast<T *>(q);
  return e;
}

static void chain_free(rd_chain *c, void *p) {
  if (!p) return;
  auto it = std::find(c->pooled.begin(), c->pooled.end(), p);
  if (it != c->pooled.end()) {
    cudaFreeAsync(p, c->st);
    c->pooled.erase(it);
  } else {
    cudaFree(p);
  }
}

// Runs f when the enclosing scope is left by an exception (not on normal returns).
struct OnThrow {
  std::function<void()> f;
  int n0 = std::uncaught_exceptions();
  ~OnThrow() {
    if (std::uncaught_exceptions() > n0 && f) f();
  }
};

// Creates a chain over the host matrix A (N x N int16 row-major, entries in [0, RD_INF]).
// Ahost == nullptr (method 1 only): the CSC comes straight from the successor generator of
// words of length m (border = App. A rules), with no dense matrix on the host or device.
static int chain_create_impl(const int16_t *Ahost, int64_t N, int m, int alpha_max, int64_t row_begin,
                             int64_t row_end, int method, void *cuda_stream, rd_chain **out, bool border = false) {
  NvtxRange nvtx_range("rd_chain_create");
  if (!out) return fail(RD_EINVAL, "rd_chain_create: out is NULL");
  *out = nullptr;
  if (method != 0 && method != 1) return fail(RD_EINVAL, "rd_chain_create: method must be 0 (dense) or 1 (structured)");
  if (method == 1 && alpha_max > kSpMaxAlpha)
    return fail(RD_EINVAL, "rd_chain_create: the structured step supports alpha_max <= %d", kSpMaxAlpha);
  if (alpha_max < 1 || alpha_max > kMaxAlpha) return fail(RD_EINVAL, "rd_chain_create: alpha_max out of 1..32");
  if (row_begin < 0 || row_end > N || row_begin >= row_end)
    return fail(RD_EINVAL, "rd_chain_create: bad row range [%lld, %lld) for N=%lld", (long long)row_begin,
                (long long)row_end, (long long)N);
  rd_chain *c = new rd_chain;
  c->m = m;
  c->method = method;
  c->alpha_max = alpha_max;
  c->N = N;
  c->r0 = row_begin;
  c->r1 = row_end;
  c->Mr = row_end - row_begin;
  c->st = (cudaStream_t)cuda_stream;
  cudaGetDevice(&c->device);
  if (method == 0) {
    c->P = round_up(N, kTile);
    c->Mp = round_up(c->Mr, kTile);
    c->slot_words = (c->P / 2) * c->Mp;
  } else {
    c->P = round_up(N, 4);          // RP pitch (u32 per row pair)
    c->Mp = round_up(c->Mr, 8);     // whole CTAs of 8 (byte kernel) or 4 rows
    c->slot_words = (c->Mp / 2) * c->P;
  }
  const int16_t *A = Ahost;
  if (A)
    for (int64_t p = c->r0; p < c->r1; ++p)
      if (A[p * N + p] < RD_INF) c->diag1 = std::min<int32_t>(c->diag1, A[p * N + p]);

  int16_t *dA = nullptr;
  auto cleanup = [&](int code) {
    chain_free(c, dA);
    chain_free(c, c->BP);
    chain_free(c, c->ring);
    chain_free(c, c->colptr);
    chain_free(c, c->ent);
    chain_free(c, c->wcol);
    chain_free(c, c->spread);
    for (void *p : {(void *)c->perm, (void *)c->inv, (void *)c->lane_col, (void *)c->slab_start, (void *)c->desc,
                    (void *)c->ent8})
      chain_free(c, p);
    delete c;
    return code;
  };
  // a host allocation that throws (std::bad_alloc in the CSC / slab builds) releases the
  // chain's device buffers on the way out; the C-ABI wrapper turns it into RD_ENOMEM
  OnThrow on_throw{[&] { cleanup(0); }};
  cudaError_t e;
  {
    // device memory first, before any host build: the ring of alpha_max + 1 powers and (dense)
    // the packed operand must fit in what the device has free
    const double need = 4.0 * (double)((alpha_max + 1) * c->slot_words) +
                        (method == 0 ? 2.0 * (double)c->P * (double)c->P : 0.0);
    size_t free_b = 0, total_b = 0;
    if ((e = cudaMemGetInfo(&free_b, &total_b)) != cudaSuccess) {
      (void)cudaGetLastError();
      return cleanup(fail(RD_ECUDA, "rd_chain_create: cudaMemGetInfo: %s", cudaGetErrorString(e)));
    }
    if (need > (double)free_b)
      return cleanup(fail(RD_ENOMEM, "rd_chain_create: needs %.1f GB of device memory (ring%s), %.1f GB free",
                          need / 1e9, method == 0 ? " + packed operand" : "", (double)free_b / 1e9));
  }
  if (method == 1) {
    c->nchunks = (int)(((N + 1) * 8 + kSpSmemMax - 1) / kSpSmemMax);
    c->Qc = (int)((N + c->nchunks - 1) / c->nchunks);   // (Qc + 1) * 8 B of shared memory
    // slab layout (g_sparse_bytes == 2): column-permuted basis, lane-per-column byte kernel
    // (below N = 2048 the step is launch-bound: the single fused 16-bit kernel is fastest,
    // m = 6: 36 vs 55 us)
    const int mode = (g_sparse_bytes == 2 && N < 2048) ? 0 : g_sparse_bytes;
    std::vector<int32_t> colptr;
    std::vector<uint32_t> ent;
    std::vector<int16_t> wcol;
    std::shared_ptr<const SlabCached> sc;
    if (!A && mode == 2) sc = slab_cached(m, border, c->nchunks, c->Qc);
    const SlabHost *S = nullptr;
    if (sc) {   // A(G) of words of length m: the host layout is built once per process
      S = &sc->S;
      for (int64_t p = c->r0; p < c->r1; ++p)
        if (sc->dg[p] < RD_INF) c->diag1 = std::min<int32_t>(c->diag1, sc->dg[p]);
      c->nnz = sc->nnz;
    } else {
      if (A) {
        build_csc(A, N, c->nchunks, c->Qc, colptr, ent);
      } else {
        std::vector<int16_t> dg;
        build_csc_direct(m, border, c->nchunks, c->Qc, colptr, ent, dg);
        for (int64_t p = c->r0; p < c->r1; ++p)
          if (dg[p] < RD_INF) c->diag1 = std::min<int32_t>(c->diag1, dg[p]);
      }
      c->nnz = colptr.back();
    }
    std::unique_ptr<SlabHost> own;
    if (!S && mode == 2) {
      own.reset(new SlabHost);
      if (build_slab_layout(N, c->nchunks, c->Qc, colptr, ent, *own)) S = own.get();
    }
    const bool slab = S != nullptr;
    const int32_t *cp_p = colptr.data();
    const uint32_t *ent_p = ent.data();
    const int16_t *wcol_p = nullptr;
    size_t cp_n = colptr.size(), ent_n = ent.size(), wcol_n = 0;
    if (slab) {
      cp_p = S->ucolptr.data(); cp_n = S->ucolptr.size();
      ent_p = S->uent.data(); ent_n = S->uent.size();
      wcol_p = S->wcol.data(); wcol_n = S->wcol.size();
      auto up = [&](void **dst, const void *src, size_t bytes) {
        if ((e = chain_malloc(c, dst, bytes)) != cudaSuccess) return false;
        return (e = cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, c->st)) == cudaSuccess;
      };
      if (!up((void **)&c->perm, S->perm.data(), S->perm.size() * 4) ||
          !up((void **)&c->inv, S->inv.data(), S->inv.size() * 4) ||
          !up((void **)&c->lane_col, S->lane_col.data(), S->lane_col.size() * 4) ||
          !up((void **)&c->slab_start, S->slab_start.data(), S->slab_start.size() * 4) ||
          !up((void **)&c->desc, S->desc.data(), S->desc.size() * 4) ||
          !up((void **)&c->ent8, S->ent8.data(), S->ent8.size() * 4))
        return cleanup(fail(RD_ENOMEM, "rd_chain_create: slab layout: %s", cudaGetErrorString(e)));
    } else {
      // uniform labels (A(G): l(q,p) depends on p only) take the byte kernel (8 rows per CTA);
      // without it, the 16-bit kernel measured faster on the general format at m = 9 (24.5 vs
      // 30.0 ms) and slower at m = 10 (762 vs 521 ms), DESIGN.md §5
      const bool want_uniform = mode || c->nchunks > 1;
      if (want_uniform && csc_to_uniform(N, c->nchunks, c->Qc, colptr, ent, wcol)) {
        cp_p = colptr.data(); cp_n = colptr.size();
        ent_p = ent.data(); ent_n = ent.size();
        wcol_p = wcol.data(); wcol_n = wcol.size();
      }
    }
    if (wcol_p) {
      if ((e = chain_malloc(c, &c->wcol, wcol_n * 2)) != cudaSuccess ||
          (e = cudaMemcpyAsync(c->wcol, wcol_p, wcol_n * 2, cudaMemcpyHostToDevice, c->st)) != cudaSuccess)
        return cleanup(fail(RD_ENOMEM, "rd_chain_create: %s", cudaGetErrorString(e)));
      if (mode) {
        int16_t mxl = 0;
        for (size_t i = 0; i < wcol_n; ++i)
          if (wcol_p[i] < RD_INF) mxl = std::max(mxl, wcol_p[i]);
        const int init[2] = {0, mxl > 254 ? 1 : 0};   // flags[1] describes A^1 (row spread <= max label)
        if ((e = chain_malloc(c, &c->spread, 8)) != cudaSuccess ||
            (e = cudaMemcpyAsync(c->spread, init, 8, cudaMemcpyHostToDevice, c->st)) != cudaSuccess ||
            (e = cudaStreamSynchronize(c->st)) != cudaSuccess)
          return cleanup(fail(RD_ENOMEM, "rd_chain_create: %s", cudaGetErrorString(e)));
      }
    }
    if ((e = chain_malloc(c, &c->colptr, cp_n * 4)) != cudaSuccess ||
        (e = chain_malloc(c, &c->ent, ent_n * 4)) != cudaSuccess ||
        (A && (e = chain_malloc(c, &dA, (size_t)(N * N * 2))) != cudaSuccess) ||
        (e = chain_malloc(c, &c->ring, (size_t)((alpha_max + 1) * c->slot_words * 4))) != cudaSuccess)
      return cleanup(fail(RD_ENOMEM, "rd_chain_create: device allocation: %s", cudaGetErrorString(e)));
    if ((e = cudaMemcpyAsync(c->colptr, cp_p, cp_n * 4, cudaMemcpyHostToDevice, c->st)) != cudaSuccess ||
        (e = cudaMemcpyAsync(c->ent, ent_p, ent_n * 4, cudaMemcpyHostToDevice, c->st)) != cudaSuccess ||
        (A && (e = cudaMemcpyAsync(dA, A, (size_t)(N * N * 2), cudaMemcpyHostToDevice, c->st)) != cudaSuccess))
      return cleanup(fail(RD_ECUDA, "rd_chain_create: H2D: %s", cudaGetErrorString(e)));
    int64_t n = (alpha_max + 1) * c->slot_words;
    fill_u32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, c->st>>>(c->ring, n, kInf2);
    if (A && !slab) {
      dim3 grid((unsigned)((c->P + 255) / 256), (unsigned)(c->Mp / 2));
      pack_rp_kernel<<<grid, 256, 0, c->st>>>(dA, N, c->Mr, N, c->r0, c->slot(1), c->P, c->Mp / 2);
    } else {
      scatter_rp_kernel<<<(unsigned)((N + 255) / 256), 256, 0, c->st>>>(c->colptr, c->ent, N, c->nchunks, c->Qc,
                                                                          c->r0, c->r1, c->slot(1), c->P, c->wcol,
                                                                          c->perm);
    }
    if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaStreamSynchronize(c->st)) != cudaSuccess)
      return cleanup(fail(RD_ECUDA, "rd_chain_create: %s", cudaGetErrorString(e)));
    chain_free(c, dA);
    dA = nullptr;
    c->k = 1;
    *out = c;
    return RD_OK;
  }
  if (!A) {
    // dense chain without a dense host matrix: CSC from the successor generator, scattered
    // into the INF-filled packed operand and A^1 panel on the device (10 MB H2D at m = 9
    // instead of 960 MB, and no N^2 host fill)
    std::vector<int32_t> colptr;
    std::vector<uint32_t> ent;
    std::vector<int16_t> dg;
    int nch = 1, qc = (int)N;
    csc_chunks_17bit(N, &nch, &qc);
    build_csc_direct(m, border, nch, qc, colptr, ent, dg);
    for (int64_t p = c->r0; p < c->r1; ++p)
      if (dg[p] < RD_INF) c->diag1 = std::min<int32_t>(c->diag1, dg[p]);
    int32_t *dcp = nullptr;
    uint32_t *dent = nullptr;
    if ((e = chain_malloc(c, &c->BP, (size_t)(c->P / 2 * c->P * 4))) != cudaSuccess ||
        (e = chain_malloc(c, &c->ring, (size_t)((alpha_max + 1) * c->slot_words * 4))) != cudaSuccess ||
        (e = chain_malloc(c, &dcp, colptr.size() * 4)) != cudaSuccess ||
        (e = chain_malloc(c, &dent, ent.size() * 4)) != cudaSuccess) {
      chain_free(c, dcp);
      return cleanup(fail(RD_ENOMEM, "rd_chain_create: device allocation: %s", cudaGetErrorString(e)));
    }
    cudaMemcpyAsync(dcp, colptr.data(), colptr.size() * 4, cudaMemcpyHostToDevice, c->st);
    cudaMemcpyAsync(dent, ent.data(), ent.size() * 4, cudaMemcpyHostToDevice, c->st);
    const int64_t nbp = c->P / 2 * c->P, nring = (alpha_max + 1) * c->slot_words;
    fill_u32_kernel<<<(unsigned)((nbp + 255) / 256), 256, 0, c->st>>>(c->BP, nbp, kInf2);
    fill_u32_kernel<<<(unsigned)((nring + 255) / 256), 256, 0, c->st>>>(c->ring, nring, kInf2);
    scatter_dense_operands_kernel<<<(unsigned)((N + 255) / 256), 256, 0, c->st>>>(dcp, dent, N, nch, qc, c->BP, c->P,
                                                                                  c->slot(1), c->Mp, c->r0, c->r1);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
    chain_free(c, dcp);
    chain_free(c, dent);
    if (e != cudaSuccess) return cleanup(fail(RD_ECUDA, "rd_chain_create: %s", cudaGetErrorString(e)));
    c->k = 1;
    *out = c;
    return RD_OK;
  }
  if ((e = chain_malloc(c, &dA, (size_t)(N * N * 2))) != cudaSuccess ||
      (e = chain_malloc(c, &c->BP, (size_t)(c->P / 2 * c->P * 4))) != cudaSuccess ||
      (e = chain_malloc(c, &c->ring, (size_t)((alpha_max + 1) * c->slot_words * 4))) != cudaSuccess)
    return cleanup(fail(RD_ENOMEM, "rd_chain_create: device allocation: %s", cudaGetErrorString(e)));
  if ((e = cudaMemcpyAsync(dA, A, (size_t)(N * N * 2), cudaMemcpyHostToDevice, c->st)) != cudaSuccess)
    return cleanup(fail(RD_ECUDA, "rd_chain_create: H2D: %s", cudaGetErrorString(e)));
  // every ring slot starts all-INF (slots are compared before they are first written)
  {
    int64_t n = (alpha_max + 1) * c->slot_words;
    fill_u32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, c->st>>>(c->ring, n, kInf2);
  }
  int rc = pack_right(dA, N, N, N, c->BP, c->P, c->P / 2, c->st);
  if (rc == RD_OK) rc = pack_left(dA, N, c->Mr, N, c->r0, c->slot(1), c->Mp, c->P / 2, c->st);
  if (rc == RD_OK && (e = cudaStreamSynchronize(c->st)) != cudaSuccess)
    rc = fail(RD_ECUDA, "rd_chain_create: %s", cudaGetErrorString(e));
  chain_free(c, dA);
  dA = nullptr;
  if (rc != RD_OK) return cleanup(rc);
  c->k = 1;
  *out = c;
  return RD_OK;
}

extern "C" int rd_chain_create_ex(int m, int alpha_max, int64_t row_begin, int64_t row_end, int method,
                                  void *cuda_stream, rd_chain **out) try {
  rd_enter();
  if (!out) return fail(RD_EINVAL, "rd_chain_create: out is NULL");
  *out = nullptr;
  // m = 12 (N = 566059): structured chains only (a dense int16 power is 641 GB)
  if (m < 1 || m > 12 || (m == 12 && method != 1))
    return fail(RD_EINVAL, "rd_chain_create: m=%d out of range (m = 12: method 1 only)", m);
  const int64_t N = count_words(m);
  // both methods: CSC from the successor generator (q-chunked where N >= 2^17), operands built
  // on the device; no dense host matrix at any order
  return chain_create_impl(nullptr, N, m, alpha_max, row_begin, row_end, method, cuda_stream, out);
} RD_ABI_CATCH("rd_chain_create_ex")

// Validates a caller's matrix: entries in [0, RD_INF] (> RD_INF is read as +inf);
// returns the largest finite entry in *maxlab.
static int check_matrix(const int16_t *A, int64_t N, int32_t *maxlab, const char *who) {
  if (!A || N < 1) return fail(RD_EINVAL, "%s: NULL matrix or N < 1", who);
  int32_t mx = 0;
  for (int64_t e = 0; e < N * N; ++e) {
    if (A[e] < 0) return fail(RD_EINVAL, "%s: negative entry at %lld (entries must be >= 0)", who, (long long)e);
    if (A[e] < RD_INF) mx = std::max<int32_t>(mx, A[e]);
  }
  *maxlab = mx;
  return RD_OK;
}

extern "C" int rd_chain_create_matrix(const int16_t *A, int64_t N, int alpha_max, int64_t row_begin,
                                      int64_t row_end, int method, void *cuda_stream, rd_chain **out) try {
  rd_enter();
  int32_t mx = 0;
  if (int rc = check_matrix(A, N, &mx, "rd_chain_create_matrix")) return rc;
  // entries above RD_INF are +inf: clamp a copy so every path sees RD_INF exactly
  std::vector<int16_t> Ac(A, A + N * N);
  for (auto &x : Ac) x = std::min<int16_t>(x, RD_INF);
  return chain_create_impl(Ac.data(), N, 0, alpha_max, row_begin, row_end, method, cuda_stream, out);
} RD_ABI_CATCH("rd_chain_create_matrix")

// Dense chain (method 0) over the packed operand of A(G) that another chain exported
// (e.g. broadcast over NVLink from rank 0): no host build, the A^1 panel comes from BP.
extern "C" int rd_chain_create_packed(int m, int alpha_max, int64_t row_begin, int64_t row_end,
                                      const uint32_t *bp_dev, int32_t diag1, void *cuda_stream, rd_chain **out) try {
  rd_enter();
  if (!out || !bp_dev) return fail(RD_EINVAL, "rd_chain_create_packed: NULL argument");
  *out = nullptr;
  if (m < 1 || m > 11) return fail(RD_EINVAL, "rd_chain_create_packed: m=%d out of range", m);
  if (alpha_max < 1 || alpha_max > kMaxAlpha) return fail(RD_EINVAL, "rd_chain_create_packed: alpha_max out of 1..32");
  const int64_t N = count_words(m);
  if (row_begin < 0 || row_end > N || row_begin >= row_end)
    return fail(RD_EINVAL, "rd_chain_create_packed: bad row range");
  rd_chain *c = new rd_chain;
  c->m = m; c->method = 0; c->alpha_max = alpha_max; c->N = N;
  c->r0 = row_begin; c->r1 = row_end; c->Mr = row_end - row_begin;
  c->st = (cudaStream_t)cuda_stream;
  cudaGetDevice(&c->device);
  c->P = round_up(N, kTile);
  c->Mp = round_up(c->Mr, kTile);
  c->slot_words = (c->P / 2) * c->Mp;
  c->diag1 = diag1;
  cudaError_t e;
  const size_t bp_bytes = (size_t)(c->P / 2 * c->P * 4);
  if ((e = chain_malloc(c, &c->BP, bp_bytes)) != cudaSuccess ||
      (e = chain_malloc(c, &c->ring, (size_t)((alpha_max + 1) * c->slot_words * 4))) != cudaSuccess) {
    rd_chain_destroy(c);
    return fail(RD_ENOMEM, "rd_chain_create_packed: %s", cudaGetErrorString(e));
  }
  if ((e = cudaMemcpyAsync(c->BP, bp_dev, bp_bytes, cudaMemcpyDeviceToDevice, c->st)) != cudaSuccess) {
    rd_chain_destroy(c);
    return fail(RD_ECUDA, "rd_chain_create_packed: %s", cudaGetErrorString(e));
  }
  const int64_t n = (alpha_max + 1) * c->slot_words;
  fill_u32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, c->st>>>(c->ring, n, kInf2);
  dim3 grid((unsigned)((c->Mp + 255) / 256), (unsigned)(c->P / 2));
  pm_from_bp_kernel<<<grid, 256, 0, c->st>>>(c->BP, c->P, c->Mr, c->r0, c->slot(1), c->Mp, c->P / 2);
  if (diag1 == INT32_MAX) {   // not supplied: the panel's self-loop labels from the packed operand
    int32_t *dd = nullptr;
    if ((e = ws_malloc((void **)&dd, 4, c->st)) == cudaSuccess) {
      int32_t init = INT32_MAX;
      cudaMemcpyAsync(dd, &init, 4, cudaMemcpyHostToDevice, c->st);
      diag_from_bp_kernel<<<(unsigned)((c->Mr + 255) / 256), 256, 0, c->st>>>(c->BP, c->P, c->r0, c->r1, dd);
      cudaMemcpyAsync(&c->diag1, dd, 4, cudaMemcpyDeviceToHost, c->st);
      cudaFreeAsync(dd, c->st);
    }
  }
  if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaStreamSynchronize(c->st)) != cudaSuccess) {
    rd_chain_destroy(c);
    return fail(RD_ECUDA, "rd_chain_create_packed: %s", cudaGetErrorString(e));
  }
  c->k = 1;
  *out = c;
  return RD_OK;
} RD_ABI_CATCH("rd_chain_create_packed")

extern "C" int rd_chain_packed_operand(const rd_chain *c, const uint32_t **bp_dev, int64_t *words) try {
  rd_enter();
  if (!c || !bp_dev || !words) return fail(RD_EINVAL, "rd_chain_packed_operand: NULL argument");
  if (c->method != 0 || !c->BP) return fail(RD_EINVAL, "rd_chain_packed_operand: not a dense chain");
  *bp_dev = c->BP;
  *words = c->P / 2 * c->P;
  return RD_OK;
} RD_ABI_CATCH("rd_chain_packed_operand")

static int g_sparse_variant = 3;
static int g_split_k_off = 0;   // rd_set_split_k(0) disables split-K for small grids
static int g_split_force = 0;   // rd_set_split_k(n >= 2): every dense step splits K n ways (probes, tests)
static int g_split_tail = 1;    // rd_set_split_tail: 0 uniform splits only, 1 model (default), 2 tail only
// rd_set_stream_k: 0 (default) off, 1 by the stage-cost model, 2 hybrid whenever the last wave is
// partial, 3 full stream-K always
static int g_stream_k = 0;
// rd_set_small_chain: dense Algorithm 2 of orders N <= kSmallMaxN as one device-resident kernel
static int g_small_chain = 1;

extern "C" int rd_set_small_chain(int enable) try {
  rd_enter();
  g_small_chain = enable ? 1 : 0;
  return RD_OK;
} RD_ABI_CATCH("rd_set_small_chain")

extern "C" int rd_set_split_tail(int mode) try {
  rd_enter();
  if (mode < 0 || mode > 2) return fail(RD_EINVAL, "rd_set_split_tail: mode must be 0, 1 or 2");
  g_split_tail = mode;
  return RD_OK;
} RD_ABI_CATCH("rd_set_split_tail")

extern "C" int rd_set_stream_k(int mode) try {
  rd_enter();
  if (mode < 0 || mode > 3) return fail(RD_EINVAL, "rd_set_stream_k: mode must be 0..3");
  g_stream_k = mode;
  return RD_OK;
} RD_ABI_CATCH("rd_set_stream_k")
// rd_set_gemm_tma: 0 = cp.async mainloop always; 1 (default) = TMA mainloop for every 128-wide
// step of >= kTmaMinStages k-stages, whole or split (measured: m = 9 1 %, m = 8
// 1.7 %, m = 9 8-rank panel with tail splits 3.9 % faster; m = 7, 40 stages, equal — round 1's
// 3-8 % loss for short CTAs no longer shows with the current kernel); 2 = TMA for every 128-wide step.
static int g_gemm_tma = 1;
constexpr int64_t kTmaMinStages = 64;

extern "C" int rd_set_gemm_tma(int mode) try {
  rd_enter();
  if (mode < 0 || mode > 3) return fail(RD_EINVAL, "rd_set_gemm_tma: mode must be 0, 1, 2 or 3");
  g_gemm_tma = mode;
  return RD_OK;
} RD_ABI_CATCH("rd_set_gemm_tma")

// The dense step's wave model (see rd_chain_step): predicted time, in 128-tile stages at full
// occupancy, of (tile width, split count); writes the best pair.  Mp = padded panel rows, P =
// padded order; tile_force 0/64/128; no_split; split_force >= 2 forces n; tma = the TMA
// mainloop is available for tn = 128, n = 1.
// tail_mode: 0 = uniform splits only, 1 = uniform or tail splits, 2 = tail splits only (n > 1)
static double dense_step_plan(int64_t Mp, int64_t P, int sms, int tile_force, int no_split, int split_force,
                              int tail_mode, bool tma, int *tn_out, int *n_out, int *tail_out) {
  static const double v128[3] = {0.0, 0.676, 1.0}, v64[4] = {0.0, 0.62, 0.90, 0.951};
  const int64_t kstages = (P / 2) / kBK2;
  // waves of `units` units of work w (in 128-tile stages) on sms x S slots
  auto waves = [&](int w_tn, int64_t units, double w) {
    const int S = w_tn == 128 ? 2 : 3;
    double t = 0.0;
    for (int64_t left = units; left > 0;) {
      const int64_t u = std::min<int64_t>(left, (int64_t)sms * S);
      left -= u;
      const int L = (int)((u + sms - 1) / sms);
      t += L * w / (w_tn == 128 ? v128[L] : v64[L]);
    }
    return t;
  };
  auto work = [&](int w_tn, int n) { return (w_tn / 128.0) * ((double)kstages / n + 1.5 + (n > 1 ? 0.2 * n : 0.0)); };
  // tail = 0: every tile split n ways; tail = 1: the whole waves unsplit, the remaining tiles
  // split n ways (< 0: not applicable)
  auto cost = [&](int w_tn, int n, int tail) {
    const int64_t tiles = (Mp / kTile) * (P / w_tn);
    double t;
    if (!tail) {
      t = waves(w_tn, tiles * n, work(w_tn, n));
    } else {
      const int64_t slots = (int64_t)sms * (w_tn == 128 ? 2 : 3);
      const int64_t full = tiles / slots * slots;
      if (full == 0 || full == tiles) return -1.0;
      t = waves(w_tn, full, work(w_tn, 1)) + waves(w_tn, (tiles - full) * n, work(w_tn, n));
    }
    if (w_tn == 128 && kstages >= kTmaMinStages && tma) t *= 0.98;   // TMA mainloop (measured 1.5-4 %)
    return t;
  };
  double best = -1.0;
  *tn_out = 128;
  *n_out = 1;
  *tail_out = 0;
  for (int w_tn : {128, 64}) {
    if (tile_force && w_tn != tile_force) continue;
    for (int n = 1; n <= 8 && (n == 1 || kstages >= 2 * n); ++n) {
      if (no_split && n > 1) break;
      if (split_force && n != std::min<int64_t>(split_force, std::max<int64_t>(1, kstages / 2))) continue;
      for (int tail = 0; tail <= (n > 1 ? 1 : 0); ++tail) {
        if (tail ? tail_mode == 0 : (tail_mode == 2 && n > 1)) continue;
        const double t = cost(w_tn, n, tail);
        if (t < 0.0) continue;
        if (best < 0.0 || t < best) { best = t; *tn_out = w_tn; *n_out = n; *tail_out = tail; }
      }
    }
  }
  return best;
}

extern "C" int rd_dense_step_plan(int64_t rows, int64_t N, int sms, int *tile, int *nsplit, int *tail, double *cost) try {
  rd_enter();
  if (rows < 1 || N < 1 || rows > N || sms < 1 || !tile || !nsplit)
    return fail(RD_EINVAL, "rd_dense_step_plan: need 1 <= rows <= N, sms >= 1, non-NULL outputs");
  int tl = 0;
  const double t = dense_step_plan(round_up(rows, kTile), round_up(N, kTile), sms, g_gemm_tile, g_split_k_off ? 1 : 0,
                                   g_split_force, g_split_tail, g_gemm_tma != 0, tile, nsplit, &tl);
  if (tail) *tail = tl;
  if (cost) *cost = t;
  return RD_OK;
} RD_ABI_CATCH("rd_dense_step_plan")


static PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    (void)cudaGetLastError();
  });
  return fn;
}

// Tensor maps of a dense chain: the ring as {Mp, P/2, alpha_max+1} u32 and the packed operand
// as {P, P/2} u32, boxes of 128 x 32 (one pipeline stage of one operand), no swizzle (the
// shared-memory layout of the cp.async path).
static int chain_tma_prepare(rd_chain *c) {
  if (c->tma_ready) return RD_OK;
  auto enc = tma_encode_fn();
  if (!enc) return fail(RD_ECUDA, "rd_chain_step: cuTensorMapEncodeTiled is unavailable");
  const cuuint64_t xd[3] = {(cuuint64_t)c->Mp, (cuuint64_t)(c->P / 2), (cuuint64_t)(c->alpha_max + 1)};
  const cuuint64_t xs[2] = {(cuuint64_t)c->Mp * 4, (cuuint64_t)c->slot_words * 4};
  const cuuint32_t box3[3] = {(cuuint32_t)kTile, (cuuint32_t)kBK2, 1}, es3[3] = {1, 1, 1};
  CUresult r = enc(&c->tma.x, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, c->ring, xd, xs, box3, es3,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(RD_ECUDA, "rd_chain_step: tensor map of the ring: CUresult %d", (int)r);
  const cuuint64_t bd[2] = {(cuuint64_t)c->P, (cuuint64_t)(c->P / 2)};
  const cuuint64_t bs[1] = {(cuuint64_t)c->P * 4};
  const cuuint32_t box2[2] = {(cuuint32_t)kTile, (cuuint32_t)kBK2}, es2[2] = {1, 1};
  r = enc(&c->tma.b, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, c->BP, bd, bs, box2, es2, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(RD_ECUDA, "rd_chain_step: tensor map of the packed operand: CUresult %d", (int)r);
  c->tma_ready = true;
  return RD_OK;
}

extern "C" int rd_set_sparse_bytes(int enable) try {
  rd_enter();
  if (enable < 0 || enable > 2) return fail(RD_EINVAL, "rd_set_sparse_bytes: 0, 1 or 2");
  g_sparse_bytes = enable;
  return RD_OK;
} RD_ABI_CATCH("rd_set_sparse_bytes")

extern "C" int rd_set_split_k(int enable) try {
  g_split_k_off = enable ? 0 : 1;
  g_split_force = enable >= 2 ? std::min(enable, 8) : 0;
  return RD_OK;
} RD_ABI_CATCH("rd_set_split_k")   // rd_set_sparse_variant (default: measured best, 1024 threads)

template <int THREADS, int UNROLL, bool UNIFORM, bool STATS = true>
static int launch_sparse_u(rd_chain *c, const SpArgs &sa, int knew, const EpiArgs &epi) {
  static bool attr_set[64] = {};
  if (c->device >= 0 && c->device < 64 && !attr_set[c->device]) {
    RD_CUDA_CHECK(cudaFuncSetAttribute(minplus_sparse_kernel<STATS, THREADS, UNROLL, UNIFORM>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kSpSmemMax));
    attr_set[c->device] = true;
  }
  minplus_sparse_kernel<STATS, THREADS, UNROLL, UNIFORM>
      <<<(unsigned)(c->Mp / 4), THREADS, (size_t)(c->Qc + 1) * 8, c->st>>>(c->slot(c->k), c->P, sa, c->slot(knew),
                                                                        epi);
  RD_CUDA_CHECK(cudaGetLastError());
  return RD_OK;
}

template <int THREADS, int UNROLL>
static int launch_sparse(rd_chain *c, const SpArgs &sa, int knew, const EpiArgs &epi) {
  return sa.wcol ? launch_sparse_u<THREADS, UNROLL, true>(c, sa, knew, epi)
                 : launch_sparse_u<THREADS, UNROLL, false>(c, sa, knew, epi);
}

// Slab-layout step: the product (byte slab kernel, or the 16-bit kernel when the current power
// spreads > 254; both launched, the other exits), then diag and the two-phase periodicity stats.
static int step_slab(rd_chain *c, int knew, EpiArgs &epi) {
  SpArgs sa{c->colptr, c->ent, c->nchunks, c->Qc, c->N, c->wcol};
  epi.spread_in = c->spread + (c->k & 1);
  epi.spread_out = c->spread + (knew & 1);
  RD_CUDA_CHECK(cudaMemsetAsync(c->spread + (knew & 1), 0, 4, c->st));
  static bool attr[64] = {};
  if (c->device >= 0 && c->device < 64 && !attr[c->device]) {
    RD_CUDA_CHECK(cudaFuncSetAttribute(minplus_slab8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kSpSmemMax + 16 * 8));
    attr[c->device] = true;
  }
  SlabArgs sb{c->desc, c->lane_col, c->ent8, c->slab_start, c->nchunks, c->Qc, c->N, c->wcol};
  minplus_slab8_kernel<<<(unsigned)(c->Mp / 8), 1024, (size_t)(c->Qc + 16) * 8, c->st>>>(
      c->slot(c->k), c->P, sb, c->slot(knew), epi.spread_in, epi.spread_out);
  RD_CUDA_CHECK(cudaGetLastError());
  EpiArgs fe = epi;
  fe.stats = nullptr;
  if (int rc = launch_sparse_u<1024, 2, true, false>(c, sa, knew, fe)) return rc;
  const uint32_t *X = c->slot(knew);
  rp_diag_kernel<<<(unsigned)((c->Mr + 255) / 256), 256, 0, c->st>>>(X, c->P, c->Mr, c->r0, c->inv, epi.stats);
  RD_CUDA_CHECK(cudaGetLastError());
  if (epi.nprev > 0) {
    PanelStatsArgs pa{};
    pa.nprev = epi.nprev;
    for (int a = 0; a < epi.nprev; ++a) pa.prev[a] = reinterpret_cast<const int16_t *>(epi.prev[a]);
    const int64_t pairs = c->Mp / 2, nb = (c->N + 127) / 128;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    // a sample of row pairs first (1/32 of the rows), then only the alphas it cannot rule out
    const bool small = pairs <= 256;
    const int stride = small ? 1 : 32;
    const int64_t np = ((pairs + 4LL * stride - 1) / (4LL * stride)) * 4;
    unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(np * nb, (int64_t)sms * 4));
    rp_stats_kernel<true><<<grid, 512, 0, c->st>>>(X, c->P, pairs, c->N, stride, pa, epi.stats);
    RD_CUDA_CHECK(cudaGetLastError());
    if (!small) {
      grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(pairs * nb, (int64_t)sms * 4));
      rp_stats_kernel<false><<<grid, 512, 0, c->st>>>(X, c->P, pairs, c->N, 1, pa, epi.stats);
      RD_CUDA_CHECK(cudaGetLastError());
    }
  }
  return RD_OK;
}

extern "C" int rd_set_sparse_variant(int v) try {
  rd_enter();
  if (v < 0 || v > 3) return fail(RD_EINVAL, "rd_set_sparse_variant: 0..3");
  g_sparse_variant = v;
  return RD_OK;
} RD_ABI_CATCH("rd_set_sparse_variant")

extern "C" int rd_chain_create(int m, int alpha_max, int64_t row_begin, int64_t row_end, void *cuda_stream,
                               rd_chain **out) try {
  return rd_chain_create_ex(m, alpha_max, row_begin, row_end, 0, cuda_stream, out);
} RD_ABI_CATCH("rd_chain_create")

extern "C" int rd_chain_destroy(rd_chain *c) try {
  if (!c) return RD_OK;
  chain_free(c, c->BP);
  chain_free(c, c->ring);
  chain_free(c, c->colptr);
  chain_free(c, c->ent);
  chain_free(c, c->wcol);
  for (cudaEvent_t &e : c->tune_ev)
    if (e) cudaEventDestroy(e);
  chain_free(c, c->ws);
  chain_free(c, c->tile_cnt);
  chain_free(c, c->spread);
  for (void *p : {(void *)c->perm, (void *)c->inv, (void *)c->lane_col, (void *)c->slab_start, (void *)c->desc,
                  (void *)c->ent8})
    chain_free(c, p);
  delete c;
  return RD_OK;
} RD_ABI_CATCH("rd_chain_destroy")

extern "C" int64_t rd_chain_order(const rd_chain *c) { return c ? c->N : -1; }
extern "C" int rd_chain_current_k(const rd_chain *c) { return c ? c->k : -1; }
extern "C" int32_t rd_chain_diag1(const rd_chain *c) { return c ? c->diag1 : INT32_MAX; }
extern "C" int rd_chain_gemm_variant(const rd_chain *c) {
  if (!c) return -1;
  return c->dpx >= 0 ? c->dpx : g_dpx_cols;
}
extern "C" double rd_chain_terms_per_step(const rd_chain *c) {
  if (!c) return -1.0;
  return c->method == 0 ? (double)c->Mr * (double)c->N * (double)c->N : (double)c->Mr * (double)c->nnz;
}

// per-tile tickets of the in-kernel fixup (split-K / stream-K), zeroed once; the kernel's last
// piece of each tile resets its counter
static int chain_tile_counters(rd_chain *c) {
  if (c->tile_cnt) return RD_OK;
  const int64_t max_tiles = (c->Mp / kTile) * (c->P / 64);
  RD_CUDA_CHECK(chain_malloc(c, &c->tile_cnt, (size_t)max_tiles * 4));
  RD_CUDA_CHECK(cudaMemsetAsync(c->tile_cnt, 0, (size_t)max_tiles * 4, c->st));
  return RD_OK;
}

extern "C" int rd_chain_step(rd_chain *c, int32_t *stats_dev) try {
  rd_enter();
  NvtxRange nvtx_range(c && c->method == 1 ? "rd_chain_step structured" : "rd_chain_step");
  if (!c || !stats_dev) return fail(RD_EINVAL, "rd_chain_step: NULL argument");
  const int knew = c->k + 1;
  EpiArgs epi{};
  epi.nprev = std::min(c->alpha_max, knew - 1);
  for (int a = 1; a <= epi.nprev; ++a) epi.prev[a - 1] = c->slot(knew - a);
  epi.stats = stats_dev;
  epi.diag_row0 = c->r0;
  stats_init_kernel<<<1, 1 + 4 * kMaxAlpha, 0, c->st>>>(stats_dev, c->alpha_max);
  RD_CUDA_CHECK(cudaGetLastError());
  if (c->method == 1 && c->ent8) {
    if (int rc = step_slab(c, knew, epi)) return rc;
    c->k = knew;
    return RD_OK;
  }
  if (c->method == 1 && c->spread) {
    // byte kernel (8 rows / CTA) unless the current power's flag says some row spreads > 254,
    // then the 16-bit kernel; both launched, the one not selected exits at once (no host sync)
    SpArgs sa{c->colptr, c->ent, c->nchunks, c->Qc, c->N, c->wcol};
    epi.spread_in = c->spread + (c->k & 1);
    epi.spread_out = c->spread + (knew & 1);
    RD_CUDA_CHECK(cudaMemsetAsync(c->spread + (knew & 1), 0, 4, c->st));
    static bool attr8[64] = {};
    if (c->device >= 0 && c->device < 64 && !attr8[c->device]) {
      RD_CUDA_CHECK(cudaFuncSetAttribute(minplus_sparse8_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kSpSmemMax));
      attr8[c->device] = true;
    }
    minplus_sparse8_kernel<true><<<(unsigned)(c->Mp / 8), 1024, (size_t)(c->Qc + 1) * 8, c->st>>>(
        c->slot(c->k), c->P, sa, c->slot(knew), epi);
    RD_CUDA_CHECK(cudaGetLastError());
    int rc1 = launch_sparse<1024, 2>(c, sa, knew, epi);
    if (rc1 != RD_OK) return rc1;
    c->k = knew;
    return RD_OK;
  }
  if (c->method == 1) {
    SpArgs sa{c->colptr, c->ent, c->nchunks, c->Qc, c->N, c->wcol};
    int rc1 = RD_OK;
    switch (g_sparse_variant) {
      case 1: rc1 = launch_sparse<512, 2>(c, sa, knew, epi); break;
      case 2: rc1 = launch_sparse<1024, 1>(c, sa, knew, epi); break;
      case 3: rc1 = launch_sparse<1024, 2>(c, sa, knew, epi); break;
      default: rc1 = launch_sparse<512, 1>(c, sa, knew, epi); break;
    }
    if (rc1 != RD_OK) return rc1;
    c->k = knew;
    return RD_OK;
  }
  // Wave model (DESIGN.md §5 "Wave quantisation"): choose the tile width tn (128: 2 CTAs/SM;
  // 64: 3 CTAs/SM, twice the tiles) and the split-K count n (k-range over n CTAs per tile,
  // in-kernel fixup) that minimise the predicted step time.  Units (tiles x n) are dispatched
  // in waves of sms x S slots; a wave whose busiest SM holds L units takes L x w / v(L), with w
  // = the unit's work in 128-tile stages (tn / 128 x (kstages / n + 1.5 fill/epilogue + 0.2 n
  // fixup)) and v(L) the SM's measured relative throughput with L resident CTAs (the issue rate
  // grows with resident warps; a 64-wide tile costs ~5% more instructions per term):
  // v128 = {0.676, 1}, v64 = {0.62, 0.90, 0.951}.  Fitted to tools/wave_probe.py
  // (profiles/r02_wave_probe.txt): it picks the measured best or within 2% for m = 6..9 and
  // row panels of 1..8 ranks.  TMA plans (tn = 128, >= kTmaMinStages stages) count 2 % faster;
  // tail splits leave the whole waves unsplit (dense_step_plan).
  //
  // Stream-K (g_stream_k): CTAs share contiguous k-stage ranges that cross tile boundaries;
  // a tile computed in pieces is finished in-kernel by its last piece (partials in c->ws,
  // tickets in c->tile_cnt).  Hybrid (mode 2): the whole waves of 128-tiles run one tile per
  // CTA and only the last partial wave's k-stages are spread over every CTA slot.  Full
  // (mode 3): every k-stage of the step is spread over the 2 x SMs CTA slots.  Mode 1 = the
  // cheaper of the wave model's plan and full stream-K by the same stage-cost model.
  const int64_t ntiles = (c->Mp / kTile) * (c->P / kTile);
  const int64_t kstages = (c->P / 2) / kBK2;
  int nsplit = 1, sk_nfull = 0, sk_nsk = 0, tn = 128, tail = 0, sms = 148;
  {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    const double best = dense_step_plan(c->Mp, c->P, sms, g_gemm_tile, g_split_k_off ? 1 : 0, g_split_force,
                                        g_split_tail, g_gemm_tma != 0, &tn, &nsplit, &tail);
    const int64_t slots = 2 * (int64_t)sms;
    const int64_t full_waves = ntiles / slots, rem = ntiles - full_waves * slots;
    if (g_stream_k == 2 && rem > 0) {
      nsplit = 1; tn = 128; tail = 0; sk_nfull = (int)(full_waves * slots);
      sk_nsk = (int)std::max<int64_t>(1, std::min<int64_t>(slots, rem * kstages / 4));   // >= 4 stages each
    } else if (g_stream_k == 3 || (g_stream_k == 1 && ntiles > 1)) {
      // full stream-K: per CTA ceil(T / slots) stages, a fill + fixup per segment (<= 3)
      const int64_t T = ntiles * kstages;
      const int nsk = (int)std::max<int64_t>(1, std::min<int64_t>(slots, T / 4));
      const double per = (double)((T + nsk - 1) / nsk);
      const double segs = std::min(3.0, 1.0 + per / (double)kstages + 1.0);
      const int L = (int)((nsk + sms - 1) / sms);   // resident CTAs on the busiest SM (<= 2)
      const double t = L * (per + 1.7 * segs) / (L == 1 ? 0.676 : 1.0);   // dense_step_plan's units
      if (g_stream_k == 3 || t < best * 0.97) {
        nsplit = 1; tn = 128; tail = 0; sk_nfull = 0; sk_nsk = nsk;
      }
    }
  }
  const TmaOps *tma = nullptr;
  if (tn == 128 && (g_gemm_tma == 2 || ((g_gemm_tma == 1 || g_gemm_tma == 3) && kstages >= kTmaMinStages))) {
    if (int rc = chain_tma_prepare(c)) return rc;
    c->tma.xslot = c->k % (c->alpha_max + 1);
    c->tma.nslots = c->alpha_max + 1;
    c->tma.refill_by_thread0 = g_gemm_tma == 3 ? 0 : 1;   // measured: the last-warp refill is no faster
    tma = &c->tma;
  }
  // The DPX/IMAD mix: d = 3 and d = 4 trade places by ~1.5 % from one B200 to the next (DESIGN.md
  // §5), so a chain of long dense steps (>= ~1 ms: ntiles x kstages >= 37000; m >= 8 and the
  // row panels of m >= 8) times brackets of four consecutive steps with d = 3, 4, 4, 3 and keeps
  // d = 4 iff its steps took less in total than the d = 3 ones (the bracket cancels the linear
  // drift of the fused stats' cost while the alpha count grows).  Steps under ~40 ms (m = 8)
  // run two brackets: their d = 3 / 4 gap (~1 %) is near the step-to-step noise.  Tuning starts
  // at the power A^4, the first whose entries are all finite (the earlier ones take the stats'
  // slow path).
  const bool tune = g_dpx_auto && sk_nsk == 0 && (double)ntiles * (double)kstages >= 37000.0 && knew >= 4;
  const int tune_steps = (double)ntiles * (double)kstages < 2.0e6 ? 8 : 4;
  static const int kTuneD[4] = {3, 4, 4, 3};
  int dpx = -1;
  if (tune && c->tune_state <= tune_steps) {
    if (c->tune_state == 0)
      for (cudaEvent_t &e : c->tune_ev) RD_CUDA_CHECK(cudaEventCreate(&e));
    if (c->tune_state < tune_steps) {
      dpx = kTuneD[c->tune_state % 4];
    } else {
      float t3 = 0.f, t4 = 0.f;
      RD_CUDA_CHECK(cudaEventSynchronize(c->tune_ev[2 * tune_steps - 1]));
      for (int i = 0; i < tune_steps; ++i) {
        float t = 0.f;
        RD_CUDA_CHECK(cudaEventElapsedTime(&t, c->tune_ev[2 * i], c->tune_ev[2 * i + 1]));
        (kTuneD[i % 4] == 4 ? t4 : t3) += t;
      }
      c->dpx = t4 < t3 ? 4 : 3;
    }
  }
  if (tune && c->tune_state >= tune_steps) dpx = c->dpx;
  const int tuning = (tune && c->tune_state < tune_steps) ? c->tune_state : -1;
  if (tuning >= 0) RD_CUDA_CHECK(cudaEventRecord(c->tune_ev[2 * tuning], c->st));
  if (sk_nsk > 0) {
    const int64_t R = (ntiles - sk_nfull) * kstages;
    const int64_t per_min = R / sk_nsk;
    const int maxseg = (int)((kstages + per_min - 1) / std::max<int64_t>(1, per_min)) + 1;
    if (!c->ws || c->nsplit < maxseg) {
      chain_free(c, c->ws);
      c->ws = nullptr;
      RD_CUDA_CHECK(chain_malloc(c, &c->ws, (size_t)maxseg * c->slot_words * 4));
      c->nsplit = maxseg;
    }
    if (int rc = chain_tile_counters(c)) return rc;
    epi.sk_nfull = sk_nfull;
    epi.sk_nsk = sk_nsk;
    epi.split_ws = c->ws;
    epi.split_stride = c->slot_words;
    epi.split_cnt = c->tile_cnt;
    int rc = launch_gemm<true, true>(c->slot(c->k), c->Mp, c->BP, c->P, c->P / 2, c->slot(knew), c->Mp, c->Mr,
                                     c->N, c->Mp, c->P, epi, c->st, 1, tma);
    if (rc != RD_OK) return rc;
  } else if (nsplit == 1) {
    int rc = launch_gemm<true, true>(c->slot(c->k), c->Mp, c->BP, c->P, c->P / 2, c->slot(knew), c->Mp, c->Mr,
                                     c->N, c->Mp, c->P, epi, c->st, 1, tma, tn, dpx);
    if (rc != RD_OK) return rc;
  } else {
    // split-K with the in-kernel fixup: partial tiles in c->ws, the last CTA of each tile folds
    // them, stores the power and computes the stats (no separate combine pass)
    if (!c->ws || c->nsplit < nsplit) {
      chain_free(c, c->ws);
      c->ws = nullptr;
      RD_CUDA_CHECK(chain_malloc(c, &c->ws, (size_t)nsplit * c->slot_words * 4));
      c->nsplit = nsplit;
    }
    if (int rc = chain_tile_counters(c)) return rc;
    epi.split_stride = c->slot_words;
    epi.split_ws = c->ws;
    epi.split_cnt = c->tile_cnt;
    if (tail) {   // the whole waves unsplit, the remaining tiles split nsplit ways
      const int64_t tiles = (c->Mp / kTile) * (c->P / tn), slots = (int64_t)sms * (tn == 128 ? 2 : 3);
      epi.tail_nfull = (int)(tiles / slots * slots);
      epi.tail_split = nsplit;
    }
    int rc = launch_gemm<true, true>(c->slot(c->k), c->Mp, c->BP, c->P, c->P / 2, c->slot(knew), c->Mp, c->Mr,
                                     c->N, c->Mp, c->P, epi, c->st, tail ? 1 : nsplit, tma, tn, dpx);
    if (rc != RD_OK) return rc;
  }
  if (tuning >= 0) RD_CUDA_CHECK(cudaEventRecord(c->tune_ev[2 * tuning + 1], c->st));
  if (tune && c->tune_state <= tune_steps) ++c->tune_state;
  c->k = knew;
  return RD_OK;
} RD_ABI_CATCH("rd_chain_step")

extern "C" int rd_panel_step(rd_chain *c, int32_t *stats_dev) try { return rd_chain_step(c, stats_dev); } RD_ABI_CATCH("rd_panel_step")

extern "C" int rd_chain_read_rows(rd_chain *c, int k, int16_t *host_out) try {
  rd_enter();
  if (!c || !host_out) return fail(RD_EINVAL, "rd_chain_read_rows: NULL argument");
  if (k < 1 || k > c->k || k < c->k - c->alpha_max)
    return fail(RD_EINVAL, "rd_chain_read_rows: power %d not in the ring (current %d)", k, c->k);
  int16_t *d = nullptr;
  RD_CUDA_CHECK(ws_malloc((void **)&d, (size_t)(c->Mr * c->N * 2), c->st));
  dim3 grid((unsigned)((c->N + 255) / 256), (unsigned)c->Mr);
  if (c->method == 0)
    unpack_pm_kernel<<<grid, 256, 0, c->st>>>(c->slot(k), c->Mp, c->Mr, c->N, d);
  else
    unpack_rp_kernel<<<grid, 256, 0, c->st>>>(c->slot(k), c->P, c->Mr, c->N, d, c->inv);
  cudaError_t e = cudaMemcpyAsync(host_out, d, (size_t)(c->Mr * c->N * 2), cudaMemcpyDeviceToHost, c->st);
  cudaFreeAsync(d, c->st);
  if (e != cudaSuccess) return fail(RD_ECUDA, "rd_chain_read_rows: %s", cudaGetErrorString(e));
  RD_CUDA_CHECK(cudaStreamSynchronize(c->st));
  return RD_OK;
} RD_ABI_CATCH("rd_chain_read_rows")

// ======================================================= peer all-gather chain ==
// The north star's all-gather form with the gather fused into the product:
// A^{k+1} = A (x) A^k (powers of A commute), rank r owns rows R_r = [b_r, b_{r+1}) of
// every power and keeps the fixed left operand A[R_r, :] (PM).  Its rows of A^k sit in its
// ring in RP layout, which is exactly the packed right-operand layout of k-pairs
// [b_r/2, b_{r+1}/2); the GEMM (OUT = kOutRP) reads every rank's slot of A^k directly through
// CUDA IPC mappings (NVLink peer memory), stage by stage, so power k+1 consumes the panels of
// power k while they stream in — no gather buffer and no separate copy.  The only
// synchronisation is the per-step stats all_reduce(MIN), which orders every rank's step k
// before any rank's step k+1 (rd.h rd_agchain_step).
struct rd_agchain {
  int m = 0, alpha_max = 0, k = 0, device = 0, world = 0, rank = 0;
  int64_t N = 0, P = 0, r0 = 0, r1 = 0, Mr = 0, Mp = 0, slot_words = 0;
  cudaStream_t st = nullptr;
  uint32_t *XL = nullptr;    // A[R_r, :] in PM layout, [P/2][Mp]
  uint32_t *ring = nullptr;  // (alpha_max+1) RP slots [Mp/2][P] of rows R_r
  int32_t diag1 = INT32_MAX;
  std::vector<int64_t> bounds;
  std::vector<const uint32_t *> peer_ring;
  std::vector<int64_t> peer_slot_words;
  std::vector<void *> ipc_mapped;
  uint32_t *slot(int kk) const { return ring + (int64_t)(kk % (alpha_max + 1)) * slot_words; }
};

extern "C" int rd_agchain_destroy(rd_agchain *c) try {
  if (!c) return RD_OK;
  for (void *p : c->ipc_mapped)
    if (p) cudaIpcCloseMemHandle(p);
  if (c->XL) cudaFree(c->XL);
  if (c->ring) cudaFree(c->ring);
  delete c;
  return RD_OK;
} RD_ABI_CATCH("rd_agchain_destroy")

extern "C" int rd_agchain_create(int m, int alpha_max, const int64_t *bounds, int world, int rank, void *cuda_stream,
                                 rd_agchain **out) try {
  rd_enter();
  NvtxRange nvtx_range("rd_agchain_create");
  if (!out || !bounds) return fail(RD_EINVAL, "rd_agchain_create: NULL argument");
  *out = nullptr;
  if (m < 1 || m > 11) return fail(RD_EINVAL, "rd_agchain_create: m=%d out of range", m);
  if (alpha_max < 1 || alpha_max > kMaxAlpha) return fail(RD_EINVAL, "rd_agchain_create: alpha_max out of 1..32");
  if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
    return fail(RD_EINVAL, "rd_agchain_create: world=%d rank=%d (world <= %d)", world, rank, kMaxPeers);
  const int64_t N = count_words(m);
  if (bounds[0] != 0 || bounds[world] != N)
    return fail(RD_EINVAL, "rd_agchain_create: bounds must run from 0 to N=%lld", (long long)N);
  for (int s = 0; s < world; ++s)
    if (bounds[s + 1] <= bounds[s] || bounds[s] % kTile != 0)
      return fail(RD_EINVAL, "rd_agchain_create: panel %d = [%lld, %lld) must be non-empty and start on a %d-row tile",
                  s, (long long)bounds[s], (long long)bounds[s + 1], kTile);
  rd_agchain *c = new rd_agchain;
  OnThrow on_throw{[&] { rd_agchain_destroy(c); }};
  c->m = m; c->alpha_max = alpha_max; c->world = world; c->rank = rank; c->N = N;
  c->bounds.assign(bounds, bounds + world + 1);
  c->r0 = bounds[rank]; c->r1 = bounds[rank + 1]; c->Mr = c->r1 - c->r0;
  c->P = round_up(N, kTile);
  c->Mp = round_up(c->Mr, kTile);
  c->slot_words = (c->Mp / 2) * c->P;
  c->st = (cudaStream_t)cuda_stream;
  c->peer_ring.assign(world, nullptr);
  c->peer_slot_words.assign(world, 0);
  c->ipc_mapped.assign(world, nullptr);
  cudaGetDevice(&c->device);
  std::vector<int32_t> colptr;
  std::vector<uint32_t> ent;
  std::vector<int16_t> dg;
  int nch = 1, qc = (int)N;
  csc_chunks_17bit(N, &nch, &qc);   // m = 11: N = 191476 >= 2^17 takes two q-chunks
  build_csc_direct(m, false, nch, qc, colptr, ent, dg);
  for (int64_t p = c->r0; p < c->r1; ++p)
    if (dg[p] < RD_INF) c->diag1 = std::min<int32_t>(c->diag1, dg[p]);
  int32_t *dcp = nullptr;
  uint32_t *dent = nullptr;
  cudaError_t e;
  // the ring is a plain cudaMalloc allocation so that cudaIpcGetMemHandle can export it
  if ((e = cudaMalloc((void **)&c->XL, (size_t)(c->P / 2 * c->Mp * 4))) != cudaSuccess ||
      (e = cudaMalloc((void **)&c->ring, (size_t)((alpha_max + 1) * c->slot_words * 4))) != cudaSuccess ||
      (e = cudaMalloc((void **)&dcp, colptr.size() * 4)) != cudaSuccess ||
      (e = cudaMalloc((void **)&dent, ent.size() * 4)) != cudaSuccess) {
    if (dcp) cudaFree(dcp);
    rd_agchain_destroy(c);
    return fail(RD_ENOMEM, "rd_agchain_create: device allocation: %s", cudaGetErrorString(e));
  }
  cudaMemcpyAsync(dcp, colptr.data(), colptr.size() * 4, cudaMemcpyHostToDevice, c->st);
  cudaMemcpyAsync(dent, ent.data(), ent.size() * 4, cudaMemcpyHostToDevice, c->st);
  const int64_t nxl = c->P / 2 * c->Mp, nring = (alpha_max + 1) * c->slot_words;
  fill_u32_kernel<<<(unsigned)((nxl + 255) / 256), 256, 0, c->st>>>(c->XL, nxl, kInf2);
  fill_u32_kernel<<<(unsigned)((nring + 255) / 256), 256, 0, c->st>>>(c->ring, nring, kInf2);
  const unsigned g = (unsigned)((N + 255) / 256);
  scatter_dense_operands_kernel<<<g, 256, 0, c->st>>>(dcp, dent, N, nch, qc, nullptr, 0, c->XL, c->Mp, c->r0, c->r1);
  scatter_rp_kernel<<<g, 256, 0, c->st>>>(dcp, dent, N, nch, qc, c->r0, c->r1, c->slot(1), c->P, nullptr, nullptr);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
  cudaFree(dcp);
  cudaFree(dent);
  if (e != cudaSuccess) {
    rd_agchain_destroy(c);
    return fail(RD_ECUDA, "rd_agchain_create: %s", cudaGetErrorString(e));
  }
  c->peer_ring[rank] = c->ring;
  c->peer_slot_words[rank] = c->slot_words;
  c->k = 1;
  *out = c;
  return RD_OK;
} RD_ABI_CATCH("rd_agchain_create")

extern "C" int rd_agchain_ipc_handle(const rd_agchain *c, void *handle_out, int64_t *slot_words) try {
  rd_enter();
  if (!c || !handle_out) return fail(RD_EINVAL, "rd_agchain_ipc_handle: NULL argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == RD_IPC_HANDLE_BYTES, "IPC handle size");
  cudaIpcMemHandle_t h;
  RD_CUDA_CHECK(cudaIpcGetMemHandle(&h, c->ring));
  memcpy(handle_out, &h, sizeof h);
  if (slot_words) *slot_words = c->slot_words;
  return RD_OK;
} RD_ABI_CATCH("rd_agchain_ipc_handle")

extern "C" int rd_agchain_ring(const rd_agchain *c, const void **ring_dev, int64_t *slot_words) try {
  rd_enter();
  if (!c || !ring_dev) return fail(RD_EINVAL, "rd_agchain_ring: NULL argument");
  *ring_dev = c->ring;
  if (slot_words) *slot_words = c->slot_words;
  return RD_OK;
} RD_ABI_CATCH("rd_agchain_ring")

extern "C" int rd_agchain_set_peer(rd_agchain *c, int s, const void *ipc_handle, const void *ring_dev,
                                   int64_t slot_words) try {
  rd_enter();
  if (!c || s < 0 || s >= c->world) return fail(RD_EINVAL, "rd_agchain_set_peer: bad chain or rank");
  if (s == c->rank) return RD_OK;
  const int64_t want = (round_up(c->bounds[s + 1] - c->bounds[s], kTile) / 2) * c->P;
  if (slot_words != want)
    return fail(RD_EINVAL, "rd_agchain_set_peer: rank %d slot has %lld words, expected %lld", s,
                (long long)slot_words, (long long)want);
  if (c->ipc_mapped[s]) {
    cudaIpcCloseMemHandle(c->ipc_mapped[s]);
    c->ipc_mapped[s] = nullptr;
  }
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof h);
    void *p = nullptr;
    RD_CUDA_CHECK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->ipc_mapped[s] = p;
    c->peer_ring[s] = reinterpret_cast<const uint32_t *>(p);
  } else {
    if (!ring_dev) return fail(RD_EINVAL, "rd_agchain_set_peer: neither an IPC handle nor a device pointer");
    // a ring on another GPU of this process is read by the GEMM directly: enable peer access
    // from the chain's device (already enabled is fine), or refuse the pointer
    cudaPointerAttributes pa{};
    RD_CUDA_CHECK(cudaPointerGetAttributes(&pa, ring_dev));
    if (pa.type != cudaMemoryTypeDevice)
      return fail(RD_EINVAL, "rd_agchain_set_peer: rank %d's ring is not device memory", s);
    if (pa.device != c->device) {
      int ok = 0;
      RD_CUDA_CHECK(cudaDeviceCanAccessPeer(&ok, c->device, pa.device));
      if (!ok)
        return fail(RD_EINVAL, "rd_agchain_set_peer: device %d cannot access rank %d's ring on device %d", c->device,
                    s, pa.device);
      int cur = 0;
      RD_CUDA_CHECK(cudaGetDevice(&cur));
      RD_CUDA_CHECK(cudaSetDevice(c->device));
      cudaError_t pe = cudaDeviceEnablePeerAccess(pa.device, 0);
      cudaSetDevice(cur);
      if (pe == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
      else if (pe != cudaSuccess)
        return fail(RD_ECUDA, "rd_agchain_set_peer: enabling peer access to device %d: %s", pa.device,
                    cudaGetErrorString(pe));
    }
    c->peer_ring[s] = reinterpret_cast<const uint32_t *>(ring_dev);
  }
  c->peer_slot_words[s] = slot_words;
  return RD_OK;
} RD_ABI_CATCH("rd_agchain_set_peer")

extern "C" int rd_agchain_step(rd_agchain *c, int32_t *stats_dev) try {
  rd_enter();
  NvtxRange nvtx_range("rd_agchain_step");
  if (!c || !stats_dev) return fail(RD_EINVAL, "rd_agchain_step: NULL argument");
  PeerB pb{};
  pb.n = c->world;
  const int ks = c->k % (c->alpha_max + 1);
  for (int s = 0; s < c->world; ++s) {
    if (!c->peer_ring[s]) return fail(RD_EINVAL, "rd_agchain_step: rank %d's ring is not set", s);
    pb.base[s] = c->peer_ring[s] + (int64_t)ks * c->peer_slot_words[s];
    pb.t0[s] = (int32_t)(c->bounds[s] / 2);
  }
  pb.t0[c->world] = (int32_t)(c->P / 2);
  const int knew = c->k + 1;
  EpiArgs epi{};
  epi.nprev = std::min(c->alpha_max, knew - 1);
  for (int a = 1; a <= epi.nprev; ++a) epi.prev[a - 1] = c->slot(knew - a);
  epi.stats = stats_dev;
  epi.diag_row0 = c->r0;
  stats_init_kernel<<<1, 1 + 4 * kMaxAlpha, 0, c->st>>>(stats_dev, c->alpha_max);
  RD_CUDA_CHECK(cudaGetLastError());
  int rc;
#define RD_AG(D) launch_gemm_v<kOutRP, true, D>(c->XL, c->Mp, nullptr, c->P, c->P / 2, c->slot(knew), c->P, c->Mr, \
                                                 c->N, c->Mp, c->P, epi, c->st, 1, pb)
  switch (g_dpx_cols) {
    case 0: rc = RD_AG(0); break;
    case 2: rc = RD_AG(2); break;
    case 3: rc = RD_AG(3); break;
    case 4: rc = RD_AG(4); break;
    default: rc = RD_AG(8); break;
  }
#undef RD_AG
  if (rc != RD_OK) return rc;
  c->k = knew;
  return RD_OK;
} RD_ABI_CATCH("rd_agchain_step")

extern "C" int rd_agchain_read_rows(rd_agchain *c, int k, int16_t *host_out) try {
  rd_enter();
  if (!c || !host_out) return fail(RD_EINVAL, "rd_agchain_read_rows: NULL argument");
  if (k < 1 || k > c->k || k < c->k - c->alpha_max)
    return fail(RD_EINVAL, "rd_agchain_read_rows: power %d not in the ring (current %d)", k, c->k);
  int16_t *d = nullptr;
  RD_CUDA_CHECK(ws_malloc((void **)&d, (size_t)(c->Mr * c->N * 2), c->st));
  dim3 grid((unsigned)((c->N + 255) / 256), (unsigned)c->Mr);
  unpack_rp_kernel<<<grid, 256, 0, c->st>>>(c->slot(k), c->P, c->Mr, c->N, d, nullptr);
  cudaError_t e = cudaMemcpyAsync(host_out, d, (size_t)(c->Mr * c->N * 2), cudaMemcpyDeviceToHost, c->st);
  cudaFreeAsync(d, c->st);
  if (e != cudaSuccess) return fail(RD_ECUDA, "rd_agchain_read_rows: %s", cudaGetErrorString(e));
  RD_CUDA_CHECK(cudaStreamSynchronize(c->st));
  return RD_OK;
} RD_ABI_CATCH("rd_agchain_read_rows")

extern "C" int32_t rd_agchain_diag1(const rd_agchain *c) { return c ? c->diag1 : INT32_MAX; }
extern "C" int64_t rd_agchain_order(const rd_agchain *c) { return c ? c->N : -1; }

// ============================================================ power sequence ==
// Argument checks shared by the power-sequence entries; maxlab = the largest label (entries
// of A^k are <= k * maxlab, R5).
static int power_sequence_check(int kmax, int alpha_max, int policy, int method, int32_t maxlab,
                                rd_period_t *out, int32_t *diag) {
  if (!out) return fail(RD_EINVAL, "rd_power_sequence: out is NULL");
  *out = rd_period_t{0, 0, 0, 0, 0};
  if (kmax < 2) return fail(RD_EINVAL, "rd_power_sequence: kmax=%d < 2", kmax);
  if (alpha_max < 1 || alpha_max > kMaxAlpha) return fail(RD_EINVAL, "rd_power_sequence: alpha_max out of range");
  if (policy != 0 && policy != 1) return fail(RD_EINVAL, "rd_power_sequence: policy must be 0 or 1");
  if (method != 0 && method != 1) return fail(RD_EINVAL, "rd_power_sequence: method must be 0 or 1");
  if ((int64_t)maxlab * kmax >= RD_INF)
    return fail(RD_ERANGE, "rd_power_sequence: max label %d x kmax %d exceeds the int16 headroom", maxlab, kmax);
  if (diag)
    for (int k = 0; k <= kmax; ++k) diag[k] = INT32_MAX;
  return RD_OK;
}

static int power_sequence_run(rd_chain *c, cudaStream_t st, int kmax, int alpha_max, int policy, int method,
                              rd_period_t *out, int32_t *diag,
                              std::chrono::steady_clock::time_point *t_done = nullptr);

extern "C" int rd_power_sequence_timed(int m, int kmax, int alpha_max, int policy, int method, rd_period_t *out,
                                       int32_t *diag, double *seconds) try {
  rd_enter();
  const auto t0 = std::chrono::steady_clock::now();
  if (m < 1 || m > 11) return fail(RD_EINVAL, "rd_power_sequence: m=%d out of range", m);
  if (int rc0 = power_sequence_check(kmax, alpha_max, policy, method, 2 * m, out, diag)) return rc0;
  const int64_t N = count_words(m);
  if (method == 0 && g_small_chain && N <= kSmallMaxN) {
    // small orders: the whole chain as one device-resident kernel (rd_small.cu)
    std::vector<int16_t> A((size_t)(N * N));
    if (int rc0 = build_matrix(m, A.data(), N)) return rc0;
    double tb = 0.0, tc = 0.0;
    const int rc = small_power_sequence(A.data(), N, kmax, alpha_max, policy, out, diag, &tb, &tc);
    if (seconds) {
      seconds[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() - tc;
      seconds[1] = tc;
    }
    return rc;
  }
  cudaStream_t st;
  RD_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  rd_chain *c = nullptr;
  int rc = rd_chain_create_ex(m, alpha_max, 0, N, method, st, &c);
  if (rc != RD_OK) { cudaStreamDestroy(st); return rc; }
  const auto t1 = std::chrono::steady_clock::now();
  auto t2 = t1;
  rc = power_sequence_run(c, st, kmax, alpha_max, policy, method, out, diag, &t2);
  if (seconds) {   // the chain ends when the decision is taken and the issued work is done
    seconds[0] = std::chrono::duration<double>(t1 - t0).count();
    seconds[1] = std::chrono::duration<double>(t2 - t1).count();
  }
  return rc;
} RD_ABI_CATCH("rd_power_sequence_timed")

extern "C" int rd_power_sequence_ex2(int m, int kmax, int alpha_max, int policy, int method, rd_period_t *out,
                                     int32_t *diag) try {
  return rd_power_sequence_timed(m, kmax, alpha_max, policy, method, out, diag, nullptr);
} RD_ABI_CATCH("rd_power_sequence_ex2")

extern "C" int rd_power_sequence_matrix(const int16_t *A, int64_t N, int kmax, int alpha_max, int policy,
                                        int method, rd_period_t *out, int32_t *diag) try {
  rd_enter();
  int32_t mx = 0;
  if (int rc0 = check_matrix(A, N, &mx, "rd_power_sequence_matrix")) return rc0;
  if (int rc0 = power_sequence_check(kmax, alpha_max, policy, method, mx, out, diag)) return rc0;
  if (method == 0 && g_small_chain && N <= kSmallMaxN) {
    std::vector<int16_t> Ac(A, A + N * N);
    for (auto &x : Ac) x = std::min<int16_t>(x, RD_INF);
    return small_power_sequence(Ac.data(), N, kmax, alpha_max, policy, out, diag, nullptr, nullptr);
  }
  cudaStream_t st;
  RD_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  rd_chain *c = nullptr;
  int rc = rd_chain_create_matrix(A, N, alpha_max, 0, N, method, st, &c);
  if (rc != RD_OK) { cudaStreamDestroy(st); return rc; }
  return power_sequence_run(c, st, kmax, alpha_max, policy, method, out, diag);
} RD_ABI_CATCH("rd_power_sequence_matrix")

// Algorithm 2's loop over a created chain (consumes c and st).
static int power_sequence_run(rd_chain *c, cudaStream_t st, int kmax, int alpha_max, int policy, int method,
                              rd_period_t *out, int32_t *diag, std::chrono::steady_clock::time_point *t_done) {
  NvtxRange nvtx_range("rd_power_sequence");
  const int64_t N = c->N;
  int rc = RD_OK;

  // Speculative depth: up to `depth` power steps are enqueued ahead of the host decision,
  // each with its own stats slot and async D2H copy, so launch and sync latency overlap the
  // GEMMs of small orders.  Steps issued past the detecting power are discarded (their
  // results are never read).  Large orders use depth 1 (dense) or 2 (structured): a step
  // there is 4-300 ms and each speculative step past the decision is wasted work.
  const int depth = method == 1 ? (N >= 7000 ? 2 : 4) : (N >= 7000 ? 1 : (N >= 2000 ? 2 : 8));
  const int slen = rd_stats_len(alpha_max);
  int32_t *dstats = nullptr, *hstats = nullptr;
  std::vector<cudaEvent_t> ev(depth, nullptr);
  cudaError_t e;
  // the pinned stats mirror is kept per thread across calls (cudaMallocHost costs ~0.1-1 ms,
  // as much as a whole small-order chain)
  static thread_local int32_t *t_hstats = nullptr;
  static thread_local size_t t_hwords = 0;
  const size_t hwords = (size_t)slen * depth;
  if (t_hwords < hwords) {
    if (t_hstats) cudaFreeHost(t_hstats);
    t_hstats = nullptr;
    t_hwords = 0;
    if ((e = cudaMallocHost((void **)&t_hstats, hwords * 4)) != cudaSuccess) {
      t_hstats = nullptr;
      rd_chain_destroy(c);
      cudaStreamDestroy(st);
      return fail(RD_ENOMEM, "rd_power_sequence: %s", cudaGetErrorString(e));
    }
    t_hwords = hwords;
  }
  hstats = t_hstats;
  cudaMemPool_t pool = chain_pool(c->device);
  if (pool) {
    if (cudaMallocFromPoolAsync((void **)&dstats, (size_t)slen * 4 * depth, pool, st) != cudaSuccess) {
      (void)cudaGetLastError();
      dstats = nullptr;
      pool = nullptr;
    }
  }
  if (!dstats && (e = cudaMalloc((void **)&dstats, (size_t)slen * 4 * depth)) != cudaSuccess) {
    rd_chain_destroy(c);
    cudaStreamDestroy(st);
    return fail(RD_ENOMEM, "rd_power_sequence: %s", cudaGetErrorString(e));
  }
  for (int q = 0; q < depth; ++q) cudaEventCreateWithFlags(&ev[q], cudaEventDisableTiming);
  if (diag) diag[1] = c->diag1;  // min_p A_pp: the self-loop labels
  int found_k = -1, n0 = 0, al = 0, be = 0, k = 1, issued = 1;
  rc = RD_OK;
  for (k = 2; k <= kmax; ++k) {
    while (issued < kmax && issued - (k - 1) < depth) {
      const int q = (issued + 1) % depth;
      if ((rc = rd_chain_step(c, dstats + q * slen)) != RD_OK) break;
      if ((e = cudaMemcpyAsync(hstats + q * slen, dstats + q * slen, (size_t)slen * 4, cudaMemcpyDeviceToHost,
                               st)) != cudaSuccess ||
          (e = cudaEventRecord(ev[q], st)) != cudaSuccess) {
        rc = fail(RD_ECUDA, "rd_power_sequence: step %d: %s", issued + 1, cudaGetErrorString(e));
        break;
      }
      ++issued;
    }
    if (rc != RD_OK) break;
    const int q = k % depth;
    if ((e = cudaEventSynchronize(ev[q])) != cudaSuccess) {
      rc = fail(RD_ECUDA, "rd_power_sequence: step %d: %s", k, cudaGetErrorString(e));
      break;
    }
    const int32_t *hs = hstats + q * slen;
    if (diag) diag[k] = hs[0] >= RD_INF ? INT32_MAX : hs[0];
    int32_t a = 0, b = 0;
    if (found_k < 0) {
      if (rd_stats_decide(hs, alpha_max, k, 0, &a, &b)) {
        found_k = k; n0 = k - a; al = a; be = b;
        if (policy == 0) break;
      }
    } else {
      int aa = k - n0;
      if (aa <= alpha_max && rd_stats_decide(hs, alpha_max, k, aa, &a, &b)) { al = a; be = b; }
      if (aa >= alpha_max) break;
    }
  }
  cudaStreamSynchronize(st);
  if (t_done) *t_done = std::chrono::steady_clock::now();
  for (int q = 0; q < depth; ++q) cudaEventDestroy(ev[q]);
  int k_stop = std::min(k, kmax);
  if (pool) cudaFreeAsync(dstats, st); else cudaFree(dstats);
  rd_chain_destroy(c);
  cudaStreamDestroy(st);
  if (rc != RD_OK) return rc;
  out->k_stop = k_stop;
  if (found_k >= 0) {
    out->found = 1; out->n0 = n0; out->alpha = al; out->beta = be;
    return RD_OK;
  }
  return RD_NOTFOUND;
}

extern "C" int rd_power_sequence_ex(int m, int kmax, int alpha_max, int policy, rd_period_t *out,
                                    int32_t *diag) try {
  return rd_power_sequence_ex2(m, kmax, alpha_max, policy, 0, out, diag);
} RD_ABI_CATCH("rd_power_sequence_ex")

extern "C" int rd_power_sequence(int m, int kmax, rd_period_t *out, int32_t *diag) try {
  return rd_power_sequence_ex(m, kmax, 10, 0, out, diag);
} RD_ABI_CATCH("rd_power_sequence")

// ================================================================ ALU probe ==
namespace {
#define RD_OPQ(x) asm volatile("" : "+r"(x))
// MODE 0: independent VIADDMNMX.S16x2 chains (the DPX issue rate).
// MODE 1: the GEMM's 8x8 accumulator tile with its default instruction mix (3 of 8
//         columns DPX, 5 via IMAD(uniform one) + VIMNMX3), operands from registers made
//         opaque each iteration: the ceiling of the mix without shared-memory traffic.
template <int MODE>
__global__ void __launch_bounds__(256, 2) alu_probe_kernel(uint32_t *sink, long long *cyc, int iters, uint32_t one) {
  long long t0 = 0, t1 = 0;
  uint32_t h = 0;
  if (MODE == 0) {
    uint32_t c[32], xa0[4], yb0[8];
    uint32_t x0 = (one ^ threadIdx.x) & 0x000F000Fu;
#pragma unroll
    for (int q = 0; q < 4; ++q) xa0[q] = x0 + q;
#pragma unroll
    for (int q = 0; q < 8; ++q) yb0[q] = x0 + 3 * q;
#pragma unroll
    for (int u = 0; u < 32; ++u) c[u] = 0x10001000u + u;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int q = 0; q < 4; ++q) RD_OPQ(xa0[q]);
#pragma unroll
      for (int q = 0; q < 8; ++q) RD_OPQ(yb0[q]);
#pragma unroll
      for (int u = 0; u < 32; ++u) c[u] = __viaddmin_s16x2(xa0[u >> 3], yb0[u & 7], c[u]);
    }
    t1 = clock64();
#pragma unroll
    for (int u = 0; u < 32; ++u) h ^= c[u];
  } else {
    uint32_t acc[8][8], x0[8], x1[8], b0[8], b1[8];
    uint32_t s = threadIdx.x * 0x00010001u;
#pragma unroll
    for (int i = 0; i < 8; ++i) { x0[i] = s + i; x1[i] = s + 2 * i; b0[i] = s + 3 * i; b1[i] = s + 5 * i; }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = kInf2;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) { RD_OPQ(x0[i]); RD_OPQ(x1[i]); RD_OPQ(b0[i]); RD_OPQ(b1[i]); }
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c < 3) {
            acc[r][c] = __viaddmin_s16x2(x0[r], b0[c], acc[r][c]);
            acc[r][c] = __viaddmin_s16x2(x1[r], b1[c], acc[r][c]);
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

template <int MODE>
int probe_one(int sms, double *minplus_per_clk_sm, double *mhz, double *instr_per_clk_sm) {
  const int blocks = sms * 2, threads = 256, iters = MODE == 0 ? 8192 : 2000;
  uint32_t *sink = nullptr;
  long long *cyc = nullptr;
  RD_CUDA_CHECK(cudaMalloc(&sink, (size_t)blocks * threads * 4));
  RD_CUDA_CHECK(cudaMalloc(&cyc, (size_t)blocks * 8));
  alu_probe_kernel<MODE><<<blocks, threads>>>(sink, cyc, 16, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  alu_probe_kernel<MODE><<<blocks, threads>>>(sink, cyc, iters, 12345);
  cudaEventRecord(e1);
  RD_CUDA_CHECK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> h(blocks);
  RD_CUDA_CHECK(cudaMemcpy(h.data(), cyc, (size_t)blocks * 8, cudaMemcpyDeviceToHost));
  long long mx = *std::max_element(h.begin(), h.end());
  // (min,+) lane-terms per thread per iteration: MODE 0 32 DPX x 2; MODE 1 64 acc x 2 k-pairs x 2
  const double terms = MODE == 0 ? 64.0 : 256.0;
  *minplus_per_clk_sm = (double)iters * terms * threads * 2 / (double)mx;
  *instr_per_clk_sm = MODE == 0 ? (double)iters * 32 * (threads / 32) * 2 / (double)mx : 0.0;
  *mhz = (double)mx / (ms * 1e3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  cudaFree(cyc);
  return RD_OK;
}
}  // namespace

extern "C" int rd_alu_probe(double out[4]) try {
  rd_enter();
  if (!out) return fail(RD_EINVAL, "rd_alu_probe: NULL");
  int dev = 0, sms = 0;
  RD_CUDA_CHECK(cudaGetDevice(&dev));
  RD_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double mp0, mhz0, ipc0, mp1, mhz1, ipc1;
  int rc = probe_one<0>(sms, &mp0, &mhz0, &ipc0);
  if (rc == RD_OK) rc = probe_one<1>(sms, &mp1, &mhz1, &ipc1);
  if (rc != RD_OK) return rc;
  out[0] = ipc0;
  out[1] = mp0;
  out[2] = mp1;
  out[3] = 0.5 * (mhz0 + mhz1);
  return RD_OK;
} RD_ABI_CATCH("rd_alu_probe")
