// Shared by the GEMM translation units of librd.so (rd_cuda.cu and rd_gemm_*.cu): tile
// constants, the device helpers of the mainloop and epilogue, the epilogue / peer / TMA argument
// blocks and the launchers of the (min,+) GEMM instances.  Not part of the C-ABI.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "rd_internal.h"

#define RD_CUDA_CHECK(expr)                                                                     \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess) return fail(RD_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                     \
  } while (0)


namespace rd {

constexpr uint32_t kInf2 = 0x3FFF3FFFu;
constexpr int kThreads = 256;
constexpr int kBK2 = 32;      // k-pairs per pipeline stage (64 k)
constexpr int kStages = 3;
constexpr int kGroup = 8;     // row-tiles per rasterisation group
constexpr int kStageWords = 2 * kBK2 * kTile;   // u32 per stage (left + right tile)
constexpr size_t kSmemBytes = (size_t)kStages * kStageWords * 4;   // 96 KB (2 CTAs/SM)

constexpr int32_t kInf32 = RD_INF32;
extern int g_raster_group;   // row-tiles per rasterisation group (rd_cuda.cu)

static __device__ __forceinline__ void stats_pair(uint32_t o, uint32_t w, uint32_t &lo2, uint32_t &hi2, uint32_t &mis,
                                           uint32_t &fin) {
  const uint32_t eo = __vcmpeq2(o, kInf2), ew = __vcmpeq2(w, kInf2);
  const uint32_t d = __vsub2(o, w);
  if (!(eo | ew)) {            // both lanes finite in both powers (every entry from k = 4 on)
    fin = 0xFFFFFFFFu;
    lo2 = __vmins2(lo2, d);
    hi2 = __vmaxs2(hi2, d);
    return;
  }
  mis |= eo ^ ew;
  const uint32_t fm = ~(eo | ew);
  fin |= fm;
  lo2 = __vmins2(lo2, (d & fm) | (0x7FFF7FFFu & ~fm));
  hi2 = __vmaxs2(hi2, (d & fm) | (0x80008000u & ~fm));
}
// --------------------------------------------------------------------- GEMM --
struct EpiArgs {
  const uint32_t *prev[kMaxAlpha];  // PM slots of A^{k+1-a}, a = 1..nprev, same ld as C
  int nprev;
  int32_t *stats;          // MIN-reducible stats vector (nullable: no stats)
  int64_t diag_row0;       // global row index of local row 0 (row panels)
  int accumulate;          // row-major output only: C = min(C, X (x) B)
  int64_t split_stride;    // split-K (gridDim.y > 1, PM output): u32 between the splits' partial tiles
  // split-K with in-kernel fixup (split_cnt != nullptr, PM output): every split CTA writes its
  // partial tile to split_ws + blockIdx.y * split_stride and takes a ticket on split_cnt[tile];
  // the last one folds the others' partials into its registers and runs the ordinary epilogue
  // (store into C, fused stats).  The counters reset themselves.
  uint32_t *split_ws;
  int *split_cnt;
  // tail split (classic CTAs, split_cnt set, tail_split >= 2): CTAs [0, tail_nfull) compute
  // whole tiles 0..tail_nfull-1 (the whole waves); the tiles after them are split tail_split
  // ways, CTA tail_nfull + u computing split u % tail_split of tile tail_nfull + u / tail_split
  int tail_nfull, tail_split;
  const int *spread_in;    // structured step: 1 if some row of X has a finite spread > 254 (nullable)
  int *spread_out;         // ... the same flag for the output, for the next step (nullable)
  // Stream-K (PM output with stats, DESIGN.md §5 "Wave quantisation"): CTAs [0, sk_nfull)
  // compute whole tiles 0..sk_nfull-1; the sk_nsk CTAs after them share the R = (ntiles -
  // sk_nfull) * KBt k-stages of the remaining tiles in equal contiguous ranges, finishing each
  // tile in-kernel through split_ws / split_cnt.  sk_nsk = 0: every CTA computes one whole tile.
  int sk_nfull, sk_nsk;
};

// Tile t of the grid in rasterised order (groups of kgroup row-tiles share right-operand
// panels in L2) -> its origin (i0, j0).
__host__ static __device__ __forceinline__ void tile_origin(int t, int nti, int ntj, int kgroup, int64_t &i0, int64_t &j0) {
  const int per_group = kgroup * ntj;
  const int g = t / per_group, first = g * kgroup;
  const int gsz = min(nti - first, kgroup);
  const int w = t - g * per_group;
  i0 = (int64_t)(first + w % gsz) * kTile;
  j0 = (int64_t)(w / gsz) * kTile;
}
// Stream-K: CTA c of nsk owns the remainder's k-stage iterations [sk_begin(c), sk_begin(c+1)).
__host__ static __device__ __forceinline__ int64_t sk_begin(int c, int64_t R, int nsk) { return R * c / nsk; }
// The CTA whose range holds iteration it.
__host__ static __device__ __forceinline__ int sk_owner(int64_t it, int64_t R, int nsk) {
  int c = (int)(it * nsk / R);
  while (c + 1 < nsk && sk_begin(c + 1, R, nsk) <= it) ++c;
  while (c > 0 && sk_begin(c, R, nsk) > it) --c;
  return c;
}

static __device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

static __device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
static __device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
static __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// mbarrier + TMA (cp.async.bulk.tensor) primitives for the TMA mainloop
static __device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
static __device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
static __device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
static __device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
static __device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "RD_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra RD_WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}
static __device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *tm, uint64_t *bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
static __device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *tm, uint64_t *bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// Tensor maps of a dense chain's operands for the TMA mainloop: X = the ring of PM slots
// ({Mp, P/2, slots} u32, box 128 x 32 x 1), B = the packed operand ({P, P/2} u32, box 128 x 32).
struct TmaOps {
  CUtensorMap x, b;
  int xslot;               // ring slot of the left operand A^k (the earlier powers: xslot - a mod nslots)
  int nslots;              // ring slots (alpha_max + 1)
  int refill_by_thread0;   // 1 (default): thread 0 waits on empty_bar, then refills; 0: the last warp to release refills
};

// One CTA computes a 128 x 128 tile of C; 256 threads in a 16 x 16 grid, each thread an
// 8 x 8 register micro-tile: rows {ty*4 + 0..3, 64 + ty*4 + 0..3}, columns
// {tx*4 + 0..3, 64 + tx*4 + 0..3}.  Per k-pair a thread reads 4 x LDS.128 and issues 64
// VIADDMNMX.S16x2 (128 (min,+) terms).  Stages of 32 k-pairs of both operands (32 KB) flow
// through a 3-deep shared-memory ring, filled either by every thread's cp.async (TMA =
// false) or, TMA = true (kOutPM only), by one thread's two cp.async.bulk.tensor copies per
// stage with mbarrier completion and per-warp release (DESIGN.md §5 "Mainloop loads").
//   OUT = kOutPM : C is PM u32 [N/2][ldc] (pairs along j), no predicates (padded).
//   OUT = kOutRow: C is row-major int16 with ldc, predicated to (M, N).
//   OUT = kOutRP : C is RP u32 [M/2][ldc] (pairs along i: C[2p][j] | C[2p+1][j] << 16), and the
//                  right operand is read straight from the ranks' memory (PeerB): k-pairs
//                  [t0[s], t0[s+1]) of B live at base[s] (the packed layout, pitch ldb), e.g.
//                  peer GPUs' ring slots mapped over NVLink (CUDA IPC).  Each stage (32 k-pairs)
//                  lies inside one rank's range (ranges are whole 128-row tiles), so the
//                  all-gather of B happens inside the mainloop's cp.async pipeline, tile by tile.
//
// Two instruction forms share the mainloop: for accumulator columns
// c < DPXC each k-pair costs one VIADDMNMX.S16x2 (alu pipe); for c >= DPXC two k-pairs
// (t, t+1) cost two packed adds s = x + b on IMAD (fma pipe; exact: lane sums <= 0x7FFE
// never carry) and one VIMNMX3.S16x2 (alu) folding both into the accumulator.  The mix
// balances the alu pipe, the fma pipe and the issue slot.  `one` is a kernel argument
// equal to 1, opaque to the compiler so that the add stays an IMAD.
// Tiles are rasterised in groups of kGroup row-tiles so CTAs resident together share
// right-operand panels in L2.
constexpr int kOutRow = 0, kOutPM = 1, kOutRP = 2;
constexpr int kMaxPeers = 16;
struct PeerB {
  const uint32_t *base[kMaxPeers];  // rank s: packed rows of B for k-pairs [t0[s], t0[s+1])
  int32_t t0[kMaxPeers + 1];
  int n;
};


// Stream-ordered device workspace from the library's pool (rd_cuda.cu).
cudaMemPool_t chain_pool(int dev);
cudaError_t ws_malloc(void **p, size_t bytes, cudaStream_t st);

// Small orders (rd_small.cu): Algorithm 2 as one device-resident cooperative kernel for the
// host matrix A (N x N int16, entries in [0, RD_INF]); times in seconds (nullable).
constexpr int kSmallMaxN = 1024;
int small_power_sequence(const int16_t *Ahost, int64_t N, int kmax, int alpha_max, int policy, rd_period_t *out,
                         int32_t *diag, double *t_build, double *t_chain);

// Launchers of the GEMM instances (defined in rd_gemm_kernels.cuh, instantiated in rd_gemm_*.cu).
template <int OUT, bool STATS, int DPXC, bool TMA = false, bool SK = false, int TN = 128>
int launch_gemm_v(const uint32_t *XT, int64_t ldx, const uint32_t *BP, int64_t ldb, int64_t kpairs, void *C,
                  int64_t ldc, int64_t M, int64_t N, int64_t Mp, int64_t Np, const EpiArgs &epi,
                  cudaStream_t st, int nsplit, const PeerB &pb, const TmaOps *tma = nullptr);
template <int DPXC>
int launch_gemm32_v(const int32_t *XT, int64_t ldx, const int32_t *BP, int64_t ldb, int64_t kp, int32_t *C,
                    int64_t ldc, int64_t M, int64_t N, int64_t Mp, int64_t Np, int accumulate, cudaStream_t st);

}  // namespace rd
