// Kernel templates of the (min,+) GEMM and their launchers; included only by the
// instantiation units rd_gemm_*.cu (compiled in parallel).  See rd_gemm.cuh.
#pragma once
#include "rd_gemm.cuh"

namespace rd {

#ifndef RD_T_UNROLL
#define RD_T_UNROLL 16   // mainloop k-pair pairs per stage: fully unrolled (A/B builds may pass -DRD_T_UNROLL)
#endif
constexpr int kTUnroll = RD_T_UNROLL;
#ifndef RD_DPX_ROW_SHIFT
#define RD_DPX_ROW_SHIFT 1   // which accumulators take the DPX form: (r * shift + r * NC + c) mod 8 < d
#endif
constexpr int kDpxRowShift = RD_DPX_ROW_SHIFT;
#ifndef RD_EPI_FAST_ALL
#define RD_EPI_FAST_ALL 1   // 0: the cp.async instances keep the next-alpha prefetch form (A/B)
#endif
constexpr bool kEpiFastAll = RD_EPI_FAST_ALL;
#ifndef RD_LOOP_CR
#define RD_LOOP_CR 0   // A/B builds: 1 visits the accumulators column-major in the stage body
#endif
#ifndef RD_STAGE_ORDER
// order of the stage body (see the mainloop): -1 (default) = order 2 for the TMA instances
// with d = 3 (m = 9 270.3 vs 278.5 ms one-pass, 272.7 two-pass), RD_STAGE_ORDER_CP (2) for the
// cp.async instances with d = 3, one pass otherwise (d = 4 is fastest in one pass:
// profiles/r02m_stage_order_ab.txt); 0..5 force an order in every instance (A/B)
#define RD_STAGE_ORDER -1
#endif
#ifndef RD_STAGE_ORDER32
#define RD_STAGE_ORDER32 2   // the 32-bit GEMM's stage body: 2 three passes (N = 7411 21.79 vs 22.25 ms one pass), 0 (A/B)
#endif
#ifndef RD_STAGE_ORDER_CP
#define RD_STAGE_ORDER_CP 2   // cp.async d = 3: m = 7 0.560 vs 0.564 ms, m = 8 11.10 vs 11.17 (profiles/r02m_stage_order_ab.txt)
#endif
#ifndef RD_DPX8_AS
#define RD_DPX8_AS 8   // A/B builds only: the d = 8 instances compile with this many DPX columns
#endif
#ifndef RD_EPI_TMA
#define RD_EPI_TMA 0   // 1: the TMA instance streams the earlier powers' tiles through the stage ring (A/B: slower)
#endif
constexpr bool kEpiTma = RD_EPI_TMA;
#ifndef RD_EPI_OPAQUE
#define RD_EPI_OPAQUE 1   // 1: the TMA epilogue re-reads `out` per alpha (nothing hoisted: no spills)
#endif

// TN = tile width (columns of C): 128 (thread tile 8 x 8, 2 CTAs/SM) or 64 (8 x 4, 3 CTAs/SM,
// twice the tiles for the same work: finer wave quantisation).  Accumulator (r, c) of a
// thread uses the DPX form when (r * NC + c) mod 8 < DPXC (TN = 128: c < DPXC), so both widths
// keep the DPXC / 8 instruction mix.
template <int OUT, bool STATS, int DPXC, bool TMA = false, bool SK = false, int TN = 128>
__global__ void __launch_bounds__(kThreads, TN == 128 ? 2 : 3)
minplus_gemm_kernel(const uint32_t *__restrict__ XT, int64_t ldx, const uint32_t *__restrict__ BP,
                    int64_t ldb, int kpairs, void *__restrict__ Cv, int64_t ldc, int64_t M, int64_t N,
                    int nti, int ntj, uint32_t one, EpiArgs epi, int kgroup, PeerB pb,
                    const __grid_constant__ TmaOps tma) {
  extern __shared__ __align__(16) uint32_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages];
  __shared__ uint32_t rel_cnt[kStages];   // TMA: warps that have released each stage
  // TMA writes need an aligned destination: the TMA variant is launched with 1 KB extra
  // dynamic shared memory and rounds its stage base up to 1 KB
  uint32_t *smem = smem_raw;
  if constexpr (TMA)
    smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) / 4u;
  const int tid = threadIdx.x;
  // a warp covers 4 (ty) x 8 (tx) threads of the 16 x 16 grid: its fragment loads touch 4 and 8
  // distinct 16-byte chunks (one shared-memory wavefront each)
  const int wq = tid >> 5, lq = tid & 31;
  const int ty = 4 * (wq >> 1) + (lq >> 3), tx = 8 * (wq & 1) + (lq & 7);
  const int KBt = kpairs / kBK2;
  constexpr int NC = TN / 16;                   // accumulator columns per thread (8 or 4)
  constexpr int SW = kBK2 * (kTile + TN);       // u32 per pipeline stage (left + right tile)
  static_assert(TN == 128 || (TN == 64 && OUT == kOutPM && !TMA && !SK), "TN = 64: PM output, cp.async");

  // cp.async mapping: the left tile is 32 k-pair rows x 32 chunks of 16 B (8 rows per pass),
  // the right tile 32 rows x TN / 4 chunks (1024 / TN rows per pass)
  const int ld_row = tid >> 5, ld_col = (tid & 31) * 4;
  constexpr int BCH = TN / 4, BRP = kThreads / BCH;
  const int ldb_row = tid / BCH, ldb_col = (tid % BCH) * 4;
  const int64_t gx_step8 = 8 * ldx;

  uint32_t acc[8][NC];
  // TMA: two bulk-tensor copies per stage (32 KB, completion counted on full_bar[s]); every
  // warp releases a consumed stage on empty_bar[s] and thread 0 refills it once all 8 warps
  // have (tma.refill_by_thread0; the alternative — the last warp to release a stage, found by a
  // shared-memory ticket, refills it and nobody waits — measured no faster).  No per-thread
  // copy instructions, no CTA-wide barrier.  Stages are
  // numbered by a running count `it` over the CTA's segments (stream-K CTAs run several), so
  // slot = it mod kStages and the barrier phases continue across segments.
  if constexpr (TMA) {
    if (tid == 0) {
#pragma unroll
      for (int s = 0; s < kStages; ++s) {
        mbar_init(&full_bar[s], 1);
        mbar_init(&empty_bar[s], kThreads / 32);
        rel_cnt[s] = 0;
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }

  // acc = min over k-stages [kb0, kb0 + KB) of the tile at (i0, j0); it0 = stages this CTA
  // consumed before (TMA slot / phase numbering)
  auto mainloop = [&](int64_t i0, int64_t j0, int kb0, int KB, uint32_t it0) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[r][c] = kInf2;
    const uint32_t *gx = XT + (int64_t)ld_row * ldx + i0 + ld_col;
    const uint32_t *gb = BP + (int64_t)ldb_row * ldb + j0 + ldb_col;
    auto load_stage = [&](int stage, int kb) {
      uint32_t *sx = smem + stage * SW;
      uint32_t *sb = sx + kBK2 * kTile;
      const int64_t ox = (int64_t)kb * kBK2 * ldx;
      const uint32_t *gbk;
      if constexpr (OUT == kOutRP) {   // the rank holding k-pairs [kb * kBK2, +kBK2)
        const int tk = kb * kBK2;
        int s = 0;
        while (s + 1 < pb.n && tk >= pb.t0[s + 1]) ++s;
        gbk = pb.base[s] + (int64_t)(tk - pb.t0[s] + ldb_row) * ldb + j0 + ldb_col;
      } else {
        gbk = gb + (int64_t)kb * kBK2 * ldb;
      }
#pragma unroll
      for (int r = 0; r < kBK2; r += 8) cp_async16(sx + (ld_row + r) * kTile + ld_col, gx + ox + (r / 8) * gx_step8);
#pragma unroll
      for (int r = 0; r < kBK2; r += BRP) cp_async16(sb + (ldb_row + r) * TN + ldb_col, gbk + (int64_t)r * ldb);
    };
    auto tma_issue = [&](int s, int kb) {
      uint32_t *sx = smem + s * SW;
      mbar_expect_tx(&full_bar[s], (uint32_t)(SW * 4));
      tma_load_3d(sx, &tma.x, &full_bar[s], (int)i0, (kb0 + kb) * kBK2, tma.xslot);
      tma_load_2d(sx + kBK2 * kTile, &tma.b, &full_bar[s], (int)j0, (kb0 + kb) * kBK2);
    };
    if constexpr (TMA) {
      if (tid == 0)
        for (int s = 0; s < kStages && s < KB; ++s) {
          const uint32_t g = it0 + s;
          if (g >= (uint32_t)kStages) mbar_wait(&empty_bar[g % kStages], ((g / kStages) - 1) & 1);
          tma_issue(g % kStages, s);
        }
    } else {
#pragma unroll
      for (int s = 0; s < kStages - 1; ++s) {
        if (s < KB) load_stage(s, kb0 + s);
        cp_async_commit();
      }
    }

    for (int kb = 0; kb < KB; ++kb) {
      const uint32_t g = it0 + kb;
      const int slot = TMA ? (int)(g % kStages) : kb % kStages;
      if constexpr (TMA) {
        mbar_wait(&full_bar[slot], (g / kStages) & 1);
      } else {
        cp_async_wait<kStages - 2>();
        __syncthreads();
        {
          int nk = kb + kStages - 1;
          if (nk < KB) load_stage(nk % kStages, kb0 + nk);
          cp_async_commit();
        }
      }
      const uint32_t *sx = smem + slot * SW;
      const uint32_t *sb = sx + kBK2 * kTile;
      if (DPXC >= 8 && RD_DPX8_AS >= 8) {
#pragma unroll
        for (int t = 0; t < kBK2; ++t) {
          const uint4 xa = *reinterpret_cast<const uint4 *>(sx + t * kTile + ty * 4);
          const uint4 xb = *reinterpret_cast<const uint4 *>(sx + t * kTile + 64 + ty * 4);
          const uint32_t x[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
          uint32_t b[NC];
#pragma unroll
          for (int h = 0; h < NC / 4; ++h) {
            const uint4 bv = *reinterpret_cast<const uint4 *>(sb + t * TN + h * 64 + tx * 4);
            b[4 * h] = bv.x; b[4 * h + 1] = bv.y; b[4 * h + 2] = bv.z; b[4 * h + 3] = bv.w;
          }
#pragma unroll
          for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[r][c] = __viaddmin_s16x2(x[r], b[c], acc[r][c]);
        }
      } else {
#pragma unroll kTUnroll
        for (int t = 0; t < kBK2; t += 2) {
          uint32_t x0[8], x1[8], b0[NC], b1[NC];
          {
            const uint4 p = *reinterpret_cast<const uint4 *>(sx + t * kTile + ty * 4);
            const uint4 q = *reinterpret_cast<const uint4 *>(sx + t * kTile + 64 + ty * 4);
            const uint4 u = *reinterpret_cast<const uint4 *>(sx + (t + 1) * kTile + ty * 4);
            const uint4 v = *reinterpret_cast<const uint4 *>(sx + (t + 1) * kTile + 64 + ty * 4);
            x0[0] = p.x; x0[1] = p.y; x0[2] = p.z; x0[3] = p.w; x0[4] = q.x; x0[5] = q.y; x0[6] = q.z; x0[7] = q.w;
            x1[0] = u.x; x1[1] = u.y; x1[2] = u.z; x1[3] = u.w; x1[4] = v.x; x1[5] = v.y; x1[6] = v.z; x1[7] = v.w;
          }
#pragma unroll
          for (int h = 0; h < NC / 4; ++h) {
            const uint4 p = *reinterpret_cast<const uint4 *>(sb + t * TN + h * 64 + tx * 4);
            const uint4 u = *reinterpret_cast<const uint4 *>(sb + (t + 1) * TN + h * 64 + tx * 4);
            b0[4 * h] = p.x; b0[4 * h + 1] = p.y; b0[4 * h + 2] = p.z; b0[4 * h + 3] = p.w;
            b1[4 * h] = u.x; b1[4 * h + 1] = u.y; b1[4 * h + 2] = u.z; b1[4 * h + 3] = u.w;
          }
          // stage-body order (RD_STAGE_ORDER): 0 = one pass, each accumulator's two k-pairs
          // together; 1 = two passes (every DPX accumulator's first k-pair, then its second with
          // the IMAD/VIMNMX3 accumulators); 2 = DPX first k-pairs, IMAD/VIMNMX3 accumulators, DPX
          // second k-pairs; 3 = IMAD/VIMNMX3 accumulators, then the DPX ones (both k-pairs);
          // 4 = 2 in two halves of rows; 5 = 2 row by row; 6 = 2 with the IMAD pass column-major;
          // 7 = 2 with the second DPX pass in reverse; 8..10 further variants of 2 (A/B).
          // Default: 2 for the instances with d = 3, else 0 (measured).
          constexpr int kOrder = RD_STAGE_ORDER >= 0 ? RD_STAGE_ORDER
                                 : DPXC != 3 ? 0 : TMA ? 2 : RD_STAGE_ORDER_CP;
          constexpr int kD = DPXC == 8 ? RD_DPX8_AS : DPXC;
          auto is_dpx = [&](int r, int c) { return (r * kDpxRowShift + r * NC + c) % 8 < kD; };
          auto dpx_k = [&](int r, int c, int h) {
            acc[r][c] = __viaddmin_s16x2(h ? x1[r] : x0[r], h ? b1[c] : b0[c], acc[r][c]);
          };
          auto imad_grp = [&](int r, int c) {
            const uint32_t s0 = x0[r] * one + b0[c];
            const uint32_t s1 = x1[r] * one + b1[c];
            acc[r][c] = __vimin3_s16x2(acc[r][c], s0, s1);
          };
          if constexpr (kOrder == 0) {
#pragma unroll
            for (int q = 0; q < 8 * NC; ++q) {
              // accumulator visit order: row-major (default) or column-major (RD_LOOP_CR, A/B)
              const int r = RD_LOOP_CR ? q % 8 : q / NC, c = RD_LOOP_CR ? q / 8 : q % NC;
              if (is_dpx(r, c)) {
                dpx_k(r, c, 0);
                dpx_k(r, c, 1);
              } else {
                imad_grp(r, c);
              }
            }
          } else if constexpr (kOrder == 1) {
#pragma unroll
            for (int q = 0; q < 8 * NC; ++q)
              if (is_dpx(q / NC, q % NC)) dpx_k(q / NC, q % NC, 0);
#pragma unroll
            for (int q = 0; q < 8 * NC; ++q) {
              if (is_dpx(q / NC, q % NC)) dpx_k(q / NC, q % NC, 1);
              else imad_grp(q / NC, q % NC);
            }
          } else if constexpr (kOrder == 2) {
#pragma unroll
            for (int q = 0; q < 8 * NC; ++q)
              if (is_dpx(q / NC, q % NC)) dpx_k(q / NC, q % NC, 0);
#pragma unroll
            for (int q = 0; q < 8 * NC; ++q)
              if (!is_dpx(q / NC, q % NC)) imad_grp(q / NC, q % NC);
#pragma unroll
            for (int q = 0; q < 8 * NC; ++q)
              if (is_dpx(q / NC, q % NC)) dpx_k(q / NC, q % NC, 1);
          } else if constexpr (kOrder == 3) {
#pragma unroll
            for (int q = 0; q < 8 * NC; ++q)
              if (!is_dpx(q / NC, q % NC)) imad_grp(q / NC, q % NC);
#pragma unroll
            for (int q = 0; q < 8 * NC; ++q)
              if (is_dpx(q / NC, q % NC)) {
                dpx_k(q / NC, q % NC, 0);
                dpx_k(q / NC, q % NC, 1);
              }
          } else if constexpr (kOrder == 4) {   // 2 in two halves of rows
#pragma unroll
            for (int q = 0; q < 8 * NC; ++q)
              if (is_dpx(q / NC, q % NC)) dpx_k(q / NC, q % NC, 0);
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
              for (int q = hh * 4 * NC; q < (hh + 1) * 4 * NC; ++q)
                if (!is_dpx(q / NC, q % NC)) imad_grp(q / NC, q % NC);
#pragma unroll
              for (int q = hh * 4 * NC; q < (hh + 1) * 4 * NC; ++q)
                if (is_dpx(q / NC, q % NC)) dpx_k(q / NC, q % NC, 1);
            }
          } else if constexpr (kOrder == 6 || kOrder == 7) {   // 2, IMAD pass column-major / DPX k1 reversed
#pragma unroll
            for (int q = 0; q < 8 * NC; ++q)
              if (is_dpx(q / NC, q % NC)) dpx_k(q / NC, q % NC, 0);
#pragma unroll
            for (int q = 0; q < 8 * NC; ++q) {
              const int r = kOrder == 6 ? q % 8 : q / NC, c = kOrder == 6 ? q / 8 : q % NC;
              if (!is_dpx(r, c)) imad_grp(r, c);
            }
#pragma unroll
            for (int q = 0; q < 8 * NC; ++q) {
              const int qq = kOrder == 7 ? 8 * NC - 1 - q : q;
              if (is_dpx(qq / NC, qq % NC)) dpx_k(qq / NC, qq % NC, 1);
            }
          } else if constexpr (kOrder >= 8 && kOrder <= 10) {
            // 8: 2 with the first DPX pass reversed; 9: 2 with the IMAD pass's rows from both ends
            // inwards; 10: 2 with the IMAD pass's columns descending
#pragma unroll
            for (int q = 0; q < 8 * NC; ++q) {
              const int qq = kOrder == 8 ? 8 * NC - 1 - q : q;
              if (is_dpx(qq / NC, qq % NC)) dpx_k(qq / NC, qq % NC, 0);
            }
#pragma unroll
            for (int q = 0; q < 8 * NC; ++q) {
              int r = q / NC, c = q % NC;
              if (kOrder == 9) r = (r & 1) ? 7 - (r >> 1) : (r >> 1);
              if (kOrder == 10) c = NC - 1 - c;
              if (!is_dpx(r, c)) imad_grp(r, c);
            }
#pragma unroll
            for (int q = 0; q < 8 * NC; ++q)
              if (is_dpx(q / NC, q % NC)) dpx_k(q / NC, q % NC, 1);
          } else {   // 2 row by row
#pragma unroll
            for (int r = 0; r < 8; ++r) {
#pragma unroll
              for (int c = 0; c < NC; ++c)
                if (is_dpx(r, c)) dpx_k(r, c, 0);
#pragma unroll
              for (int c = 0; c < NC; ++c)
                if (!is_dpx(r, c)) imad_grp(r, c);
#pragma unroll
              for (int c = 0; c < NC; ++c)
                if (is_dpx(r, c)) dpx_k(r, c, 1);
            }
          }
        }
      }
      if constexpr (TMA) {   // release this stage; the last warp to release it refills it
        __syncwarp();
        if (tma.refill_by_thread0) {   // thread 0 waits for every warp, then refills
          if ((tid & 31) == 0) mbar_arrive(&empty_bar[slot]);
          if (tid == 0 && kb + kStages < KB) {
            mbar_wait(&empty_bar[slot], (g / kStages) & 1);
            tma_issue(slot, kb + kStages);
          }
        } else if ((tid & 31) == 0) {
          mbar_arrive(&empty_bar[slot]);   // phase bookkeeping for later segments' prologues
          if (atomicAdd(&rel_cnt[slot], 1u) == kThreads / 32 - 1) {
            rel_cnt[slot] = 0;
            if (kb + kStages < KB) tma_issue(slot, kb + kStages);
          }
        }
      }
    }
    if constexpr (!TMA) cp_async_wait<0>();
  };

  // ---------------------------------------------------------------- epilogue --
  // v = min(lo, hi) per accumulator; pairs (c, c+1) packed (min_c | min_{c+1} << 16).
  uint32_t out[8][NC / 2];
  auto fold = [&]() {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int p = 0; p < NC / 2; ++p) {
        uint32_t a0 = acc[r][2 * p], a1 = acc[r][2 * p + 1];
        out[r][p] = __vmins2(prmt(a0, a1, 0x5410), prmt(a0, a1, 0x7632));
      }
  };
  // PM store of the folded tile at (i0, j0) into C (pitch ldc)
  auto store_pm = [&](uint32_t *C, int64_t i0, int64_t j0) {
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
      for (int p = 0; p < NC / 2; ++p) {
        // column pair jp covers columns j0 + (p>>1)*64 + tx*4 + (p&1)*2 + {0,1}
        int64_t jp = (j0 + (p >> 1) * 64 + tx * 4 + (p & 1) * 2) >> 1;
        uint4 v = make_uint4(out[g * 4 + 0][p], out[g * 4 + 1][p], out[g * 4 + 2][p], out[g * 4 + 3][p]);
        *reinterpret_cast<uint4 *>(C + jp * ldc + i0 + g * 64 + ty * 4) = v;
      }
  };

  // Work units.  Classic CTA: one whole tile (split-K: the k-range blockIdx.y of gridDim.y).
  // Stream-K CTA (SK, blockIdx.x >= sk_nfull): an equal contiguous share of the remaining
  // tiles' k-stages, walked segment by segment (a segment = the part of the range inside one
  // tile).  A tile computed in several pieces (split-K splits or stream-K segments) is finished
  // in-kernel: every piece stores its partial tile to split_ws + seg * split_stride and takes a
  // ticket on split_cnt[tile]; the last one folds the others' partials into its registers and
  // runs the ordinary epilogue (store into C, fused stats).  The counters reset themselves.
  __shared__ int s_last;
  __shared__ int32_t red[kThreads / 32][1 + 4 * kMaxAlpha];
  int64_t i0, j0;
  const bool skc = SK && (int)blockIdx.x >= epi.sk_nfull;
  int64_t ke = 0, ke1 = 0, R = 0;
  int skid = 0;
  if (skc) {
    skid = (int)blockIdx.x - epi.sk_nfull;
    R = (int64_t)(nti * ntj - epi.sk_nfull) * KBt;
    ke = sk_begin(skid, R, epi.sk_nsk);
    ke1 = sk_begin(skid + 1, R, epi.sk_nsk);
  }
  uint32_t it = 0;
  for (;;) {
    int kb0, KB, seg, nseg, tile;
    if (skc) {
      if (ke >= ke1) return;
      const int r = (int)(ke / KBt);
      kb0 = (int)(ke - (int64_t)r * KBt);
      KB = (int)((ke1 - ke) < (int64_t)(KBt - kb0) ? (ke1 - ke) : (int64_t)(KBt - kb0));
      const int own0 = sk_owner((int64_t)r * KBt, R, epi.sk_nsk);
      seg = skid - own0;
      nseg = sk_owner((int64_t)r * KBt + KBt - 1, R, epi.sk_nsk) - own0 + 1;
      tile = epi.sk_nfull + r;
      tile_origin(tile, nti, ntj, kgroup, i0, j0);   // SK: TN = 128
      if (it > 0 && !TMA) __syncthreads();   // every warp is done with the previous segment's stages
    } else {
      tile = (int)blockIdx.x;
      seg = (int)blockIdx.y;
      nseg = (int)gridDim.y;
      if (epi.tail_split > 1 && tile >= epi.tail_nfull) {   // a split of a tail tile
        const int u = tile - epi.tail_nfull;
        tile = epi.tail_nfull + u / epi.tail_split;
        seg = u - (tile - epi.tail_nfull) * epi.tail_split;
        nseg = epi.tail_split;
      }
      tile_origin(tile, nti, ntj, kgroup, i0, j0);
      if constexpr (TN != kTile) j0 = j0 / kTile * TN;
      kb0 = (int)((int64_t)KBt * seg / nseg);
      KB = (int)((int64_t)KBt * (seg + 1) / nseg) - kb0;
    }
    mainloop(i0, j0, kb0, KB, it);
    it += (uint32_t)KB;
    ke += KB;
    fold();
    bool fixed_up = false;
    if constexpr (OUT == kOutPM && STATS) {
      if (nseg > 1 && epi.split_cnt) {   // the last piece of the tile finishes it
        store_pm(epi.split_ws + (int64_t)seg * epi.split_stride, i0, j0);
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = atomicAdd(&epi.split_cnt[tile], 1) == nseg - 1;
        __syncthreads();
        if (!s_last) {
          if (skc) continue;
          return;
        }
        __threadfence();
        for (int sp = 0; sp < nseg; ++sp) {
          if (sp == seg) continue;
          const uint32_t *W = epi.split_ws + (int64_t)sp * epi.split_stride;
#pragma unroll
          for (int g = 0; g < 2; ++g)
#pragma unroll
            for (int p = 0; p < NC / 2; ++p) {
              const int64_t jp = (j0 + (p >> 1) * 64 + tx * 4 + (p & 1) * 2) >> 1;
              const uint4 w = __ldcg(reinterpret_cast<const uint4 *>(W + jp * ldc + i0 + g * 64 + ty * 4));
              out[g * 4 + 0][p] = __vmins2(out[g * 4 + 0][p], w.x);
              out[g * 4 + 1][p] = __vmins2(out[g * 4 + 1][p], w.y);
              out[g * 4 + 2][p] = __vmins2(out[g * 4 + 2][p], w.z);
              out[g * 4 + 3][p] = __vmins2(out[g * 4 + 3][p], w.w);
            }
        }
        if (tid == 0) epi.split_cnt[tile] = 0;   // ready for the next step
        fixed_up = true;
      }
    }

  // RP word (rows 2q', 2q'+1 of row group g; columns h*64 + tx*4 + e) from the folded pairs
  auto rp_word = [&](int g, int q, int h, int e) -> uint32_t {
    const uint32_t a = out[g * 4 + 2 * q][2 * h + (e >> 1)], b = out[g * 4 + 2 * q + 1][2 * h + (e >> 1)];
    return prmt(a, b, (e & 1) ? 0x7632 : 0x5410);
  };
  if constexpr (OUT == kOutRP) {
    uint32_t *C = reinterpret_cast<uint32_t *>(Cv);
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t pr = ((i0 + g * 64 + ty * 4) >> 1) + q;
          const uint4 v = make_uint4(rp_word(g, q, h, 0), rp_word(g, q, h, 1), rp_word(g, q, h, 2), rp_word(g, q, h, 3));
          *reinterpret_cast<uint4 *>(C + pr * ldc + j0 + h * 64 + tx * 4) = v;
        }
  } else if constexpr (OUT == kOutPM) {
    store_pm(reinterpret_cast<uint32_t *>(Cv) + (fixed_up ? 0 : (int64_t)blockIdx.y * epi.split_stride), i0, j0);
  } else {
    int16_t *C = reinterpret_cast<int16_t *>(Cv);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      int64_t i = i0 + (r >> 2) * 64 + ty * 4 + (r & 3);
      if (i >= M) continue;
#pragma unroll
      for (int p = 0; p < NC / 2; ++p) {
        int64_t j = j0 + (p >> 1) * 64 + tx * 4 + (p & 1) * 2;
        int v0 = (int)(out[r][p] & 0xFFFF), v1 = (int)(out[r][p] >> 16);
        if (epi.accumulate) {
          if (j < N) v0 = min(v0, min((int)C[i * ldc + j], (int)RD_INF));
          if (j + 1 < N) v1 = min(v1, min((int)C[i * ldc + j + 1], (int)RD_INF));
        }
        if (j < N) C[i * ldc + j] = (int16_t)v0;
        if (j + 1 < N) C[i * ldc + j + 1] = (int16_t)v1;
      }
    }
  }

  if (!STATS) return;

  // ---- fused reductions over this tile (MIN-reducible; see rd.h rd_chain_step) ----
  const int warp = tid >> 5, lane = tid & 31;

  // diagonal min (Cor 7): global row diag_row0 + i == column j
  int32_t dmin = INT_MAX;
  {
    const int64_t gi0 = epi.diag_row0 + i0;
    if (gi0 < j0 + TN && j0 < gi0 + kTile) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int p = 0; p < NC / 2; ++p)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            int64_t gi = gi0 + (r >> 2) * 64 + ty * 4 + (r & 3);
            int64_t j = j0 + (p >> 1) * 64 + tx * 4 + (p & 1) * 2 + h;
            int32_t v = (int32_t)((out[r][p] >> (16 * h)) & 0xFFFF);
            if (gi == j && v < dmin) dmin = v;
          }
    }
  }
  dmin = __reduce_min_sync(0xffffffffu, dmin);
  if (lane == 0) red[warp][0] = dmin;

  // periodicity stats against A^{k+1-a}: same PM address in the previous slots
  uint4 pv[2][NC / 2];
  uint32_t out_inf = 0;   // some lane of this thread's output is inf (the fast path's test)
  if constexpr (TMA || kEpiFastAll) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int p = 0; p < NC / 2; ++p) out_inf |= __vcmpeq2(out[r][p], kInf2);
  }
  // TMA instance: the earlier powers' tiles (A^{k+1-a} at this tile's PM address: 64 column
  // pairs x 128 rows = two 32 x 128 boxes of the ring's tensor map, 32 KB = one stage) stream
  // through the freed stage ring, numbered after the mainloop's stages so the full / empty
  // barrier phases carry on; thread 0 issues them as the warps release the stages.
  constexpr bool kStream = TMA && kEpiTma && OUT == kOutPM;
  auto epi_issue = [&](int a) {
    const uint32_t g = it + (uint32_t)a;
    const int s = (int)(g % kStages);
    if (g >= (uint32_t)kStages) mbar_wait(&empty_bar[s], ((g / kStages) - 1) & 1);
    uint32_t *dst = smem + s * SW;
    const int sl = (tma.xslot - a + tma.nslots) % tma.nslots;
    mbar_expect_tx(&full_bar[s], (uint32_t)(SW * 4));
    tma_load_3d(dst, &tma.x, &full_bar[s], (int)i0, (int)(j0 / 2), sl);
    tma_load_3d(dst + kBK2 * kTile, &tma.x, &full_bar[s], (int)i0, (int)(j0 / 2) + kBK2, sl);
  };
  if constexpr (kStream) {
    if (tid == 0)
      for (int a = 0; a < kStages && a < epi.nprev; ++a) epi_issue(a);
  }
  if constexpr (OUT != kOutRP && !kStream) {
    if (epi.nprev > 0) {
#pragma unroll
      for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int p = 0; p < NC / 2; ++p) {
          const int64_t jp = (j0 + (p >> 1) * 64 + tx * 4 + (p & 1) * 2) >> 1;
          pv[g][p] = __ldg(reinterpret_cast<const uint4 *>(epi.prev[0] + jp * ldc + i0 + g * 64 + ty * 4));
        }
    }
  }
  for (int a = 0; a < epi.nprev; ++a) {
    const uint32_t *P = epi.prev[a];
    uint32_t lo2 = 0x7FFF7FFFu, hi2 = 0x80008000u, mis = 0, fin = 0;
    if constexpr (OUT == kOutRP) {
#pragma unroll
      for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t pr = ((i0 + g * 64 + ty * 4) >> 1) + q;
            const uint4 pv = __ldg(reinterpret_cast<const uint4 *>(P + pr * ldc + j0 + h * 64 + tx * 4));
            const uint32_t pw[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) stats_pair(rp_word(g, q, h, e), pw[e], lo2, hi2, mis, fin);
          }
    } else if constexpr (TMA || kEpiFastAll) {
      // one load batch per alpha and an all-finite fast path, `out` kept opaque per alpha
      // (RD_EPI_OPAQUE).  Without the opaque marks this form cost the cp.async instances 4.6 %
      // (profiles/r02i_epilogue_fastpath_ab.txt); with them it gains 1.0 % (TMA, m = 9) and
      // 1.1 % (cp.async, m = 8): profiles/r02l_epi_opaque_ab.txt, r02l_epi_fastall_ab.txt
      if constexpr (kStream) {
        const uint32_t g = it + (uint32_t)a;
        const int s = (int)(g % kStages);
        mbar_wait(&full_bar[s], (g / kStages) & 1);
        const uint32_t *T = smem + s * SW;
#pragma unroll
        for (int g2 = 0; g2 < 2; ++g2)
#pragma unroll
          for (int p = 0; p < NC / 2; ++p)
            pv[g2][p] = *reinterpret_cast<const uint4 *>(T + ((p >> 1) * 32 + tx * 2 + (p & 1)) * kTile + g2 * 64 + ty * 4);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[s]);
        if (tid == 0 && a + kStages < epi.nprev) epi_issue(a + kStages);
      } else if (a > 0) {
        const uint32_t *Pa = epi.prev[a];
        const int64_t ldc_a = ldc;
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
          for (int p = 0; p < NC / 2; ++p) {
            const int64_t jp = (j0 + (p >> 1) * 64 + tx * 4 + (p & 1) * 2) >> 1;
            pv[g][p] = __ldg(reinterpret_cast<const uint4 *>(Pa + jp * ldc_a + i0 + g * 64 + ty * 4));
          }
      }
#if RD_EPI_OPAQUE
      // keep ptxas from hoisting the slow path's per-word inf masks of `out` out of the alpha
      // loop (32 loop-invariant registers, spilled at the 128-register cap)
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int p = 0; p < NC / 2; ++p) asm volatile("" : "+r"(out[r][p]));
#endif
      // all-finite fast path (every power from k = 4 on): one inf test over this alpha's chunks,
      // then 3 instructions per word instead of stats_pair's 8
      uint32_t iw = out_inf;
#pragma unroll
      for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int p = 0; p < NC / 2; ++p)
          iw |= __vcmpeq2(pv[g][p].x, kInf2) | __vcmpeq2(pv[g][p].y, kInf2) | __vcmpeq2(pv[g][p].z, kInf2) |
                __vcmpeq2(pv[g][p].w, kInf2);
      if (iw == 0) {
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
          for (int p = 0; p < NC / 2; ++p) {
            const uint32_t pw[4] = {pv[g][p].x, pv[g][p].y, pv[g][p].z, pv[g][p].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint32_t d = __vsub2(out[g * 4 + q][p], pw[q]);
              lo2 = __vmins2(lo2, d);
              hi2 = __vmaxs2(hi2, d);
            }
          }
        fin = 0xFFFFFFFFu;
      } else {
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
          for (int p = 0; p < NC / 2; ++p) {
            const uint32_t pw[4] = {pv[g][p].x, pv[g][p].y, pv[g][p].z, pv[g][p].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) stats_pair(out[g * 4 + q][p], pw[q], lo2, hi2, mis, fin);
          }
      }
    } else {
      // this alpha's chunks were fetched during the previous alpha (pv); fetch the next ones
      // before folding these, so the earlier powers' loads overlap the reductions
      uint4 nx[2][NC / 2];
      if (a + 1 < epi.nprev) {
        const uint32_t *Pn = epi.prev[a + 1];
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
          for (int p = 0; p < NC / 2; ++p) {
            const int64_t jp = (j0 + (p >> 1) * 64 + tx * 4 + (p & 1) * 2) >> 1;
            nx[g][p] = __ldg(reinterpret_cast<const uint4 *>(Pn + jp * ldc + i0 + g * 64 + ty * 4));
          }
      }
#pragma unroll
      for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int p = 0; p < NC / 2; ++p) {
          const uint32_t pw[4] = {pv[g][p].x, pv[g][p].y, pv[g][p].z, pv[g][p].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) stats_pair(out[g * 4 + q][p], pw[q], lo2, hi2, mis, fin);
        }
#pragma unroll
      for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int p = 0; p < NC / 2; ++p) pv[g][p] = nx[g][p];
    }
    int32_t lo = min((int32_t)(int16_t)(lo2 & 0xFFFF), (int32_t)(int16_t)(lo2 >> 16));
    int32_t hi = max((int32_t)(int16_t)(hi2 & 0xFFFF), (int32_t)(int16_t)(hi2 >> 16));
    if (!(fin & 0xFFFF) && !(fin >> 16)) { lo = INT_MAX; hi = INT_MIN + 1; }
    int32_t v0 = __reduce_min_sync(0xffffffffu, lo);
    int32_t v1 = __reduce_min_sync(0xffffffffu, -hi);
    int32_t v2 = __reduce_min_sync(0xffffffffu, mis ? -1 : 0);
    int32_t v3 = __reduce_min_sync(0xffffffffu, fin ? -1 : 0);
    if (lane == 0) {
      red[warp][1 + 4 * a + 0] = v0;
      red[warp][1 + 4 * a + 1] = v1;
      red[warp][1 + 4 * a + 2] = v2;
      red[warp][1 + 4 * a + 3] = v3;
    }
  }
  if constexpr (kStream) it += (uint32_t)epi.nprev;   // the epilogue's stages
  __syncthreads();
  const int nval = 1 + 4 * epi.nprev;
  for (int e = tid; e < nval; e += kThreads) {
    int32_t v = red[0][e];
#pragma unroll
    for (int w = 1; w < kThreads / 32; ++w) v = min(v, red[w][e]);
    atomicMin(epi.stats + e, v);
  }
  if (!skc) return;
  __syncthreads();   // red[] and the stage buffers are reused by the next segment
  }
}

// ----------------------------------------------------------- 32-bit GEMM --
// The generic product for entries beyond the int16 headroom (the
// `__viaddmin_s32` variant; rd.h rd_minplus_mul32).  Same CTA tile, thread tile, cp.async
// pipeline and rasterisation as minplus_gemm_kernel, one int32 per k instead of a k-pair:
//   XT[k][i] = X[i][k]  (left operand transposed, [Kp][Mp]),  BP[k][j] = B[k][j]  ([Kp][Np]),
// both INF32-padded to the tile, entries clamped to [., RD_INF32] on packing.  Per k a thread
// reads 4 x LDS.128 and updates 64 accumulators: columns c < DPXC with one VIADDMNMX (32-bit,
// alu), the others two k at a time with two IMAD adds (fma; exact: sums <= 0x7FFFFFFE) and one
// VIMNMX3 (alu).  RD_INF32 + anything >= RD_INF32, and accumulators start at RD_INF32, so
// infinite results come out exactly RD_INF32 (finite sums >= RD_INF32 saturate to it).

template <int DPXC>
__global__ void __launch_bounds__(kThreads, 2)
minplus_gemm32_kernel(const int32_t *__restrict__ XT, int64_t ldx, const int32_t *__restrict__ BP, int64_t ldb,
                      int kp, int32_t *__restrict__ C, int64_t ldc, int64_t M, int64_t N, int nti, int ntj,
                      int32_t one, int accumulate, int kgroup) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int tid = threadIdx.x;
  const int wq = tid >> 5, lq = tid & 31;
  const int ty = 4 * (wq >> 1) + (lq >> 3), tx = 8 * (wq & 1) + (lq & 7);
  int64_t i0, j0;
  {
    const int bid = blockIdx.x;
    const int per_group = kgroup * ntj;
    const int g = bid / per_group, first = g * kgroup;
    const int gsz = min(nti - first, kgroup);
    const int w = bid - g * per_group;
    i0 = (int64_t)(first + w % gsz) * kTile;
    j0 = (int64_t)(w / gsz) * kTile;
  }
  const int ld_row = tid >> 5, ld_col = (tid & 31) * 4;
  const int32_t *gx = XT + (int64_t)ld_row * ldx + i0 + ld_col;
  const int32_t *gb = BP + (int64_t)ld_row * ldb + j0 + ld_col;
  auto load_stage = [&](int stage, int kb) {
    uint32_t *sx = smem + stage * kStageWords;
    uint32_t *sb = sx + kBK2 * kTile;
    const int64_t ox = (int64_t)kb * kBK2 * ldx, ob = (int64_t)kb * kBK2 * ldb;
#pragma unroll
    for (int r = 0; r < kBK2; r += 8) {
      cp_async16(sx + (ld_row + r) * kTile + ld_col, gx + ox + (r / 8) * 8 * ldx);
      cp_async16(sb + (ld_row + r) * kTile + ld_col, gb + ob + (r / 8) * 8 * ldb);
    }
  };
  int32_t acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = kInf32;
  const int KB = kp / kBK2;
#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) {
    if (st < KB) load_stage(st, st);
    cp_async_commit();
  }
  for (int kb = 0; kb < KB; ++kb) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    {
      const int nk = kb + kStages - 1;
      if (nk < KB) load_stage(nk % kStages, nk);
      cp_async_commit();
    }
    const int32_t *sx = reinterpret_cast<const int32_t *>(smem + (kb % kStages) * kStageWords);
    const int32_t *sb = sx + kBK2 * kTile;
#pragma unroll
    for (int t = 0; t < kBK2; t += 2) {
      int32_t x0[8], x1[8], b0[8], b1[8];
      {
        const int4 p = *reinterpret_cast<const int4 *>(sx + t * kTile + ty * 4);
        const int4 q = *reinterpret_cast<const int4 *>(sx + t * kTile + 64 + ty * 4);
        const int4 u = *reinterpret_cast<const int4 *>(sx + (t + 1) * kTile + ty * 4);
        const int4 v = *reinterpret_cast<const int4 *>(sx + (t + 1) * kTile + 64 + ty * 4);
        x0[0] = p.x; x0[1] = p.y; x0[2] = p.z; x0[3] = p.w; x0[4] = q.x; x0[5] = q.y; x0[6] = q.z; x0[7] = q.w;
        x1[0] = u.x; x1[1] = u.y; x1[2] = u.z; x1[3] = u.w; x1[4] = v.x; x1[5] = v.y; x1[6] = v.z; x1[7] = v.w;
      }
      {
        const int4 p = *reinterpret_cast<const int4 *>(sb + t * kTile + tx * 4);
        const int4 q = *reinterpret_cast<const int4 *>(sb + t * kTile + 64 + tx * 4);
        const int4 u = *reinterpret_cast<const int4 *>(sb + (t + 1) * kTile + tx * 4);
        const int4 v = *reinterpret_cast<const int4 *>(sb + (t + 1) * kTile + 64 + tx * 4);
        b0[0] = p.x; b0[1] = p.y; b0[2] = p.z; b0[3] = p.w; b0[4] = q.x; b0[5] = q.y; b0[6] = q.z; b0[7] = q.w;
        b1[0] = u.x; b1[1] = u.y; b1[2] = u.z; b1[3] = u.w; b1[4] = v.x; b1[5] = v.y; b1[6] = v.z; b1[7] = v.w;
      }
      if constexpr (RD_STAGE_ORDER32 == 2) {   // DPX first k | IMAD/VIMNMX3 | DPX second k (A/B)
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < DPXC; ++c) acc[r][c] = __viaddmin_s32(x0[r], b0[c], acc[r][c]);
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = DPXC; c < 8; ++c) {
            const int32_t s0 = x0[r] * one + b0[c];
            const int32_t s1 = x1[r] * one + b1[c];
            acc[r][c] = __vimin3_s32(acc[r][c], s0, s1);
          }
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < DPXC; ++c) acc[r][c] = __viaddmin_s32(x1[r], b1[c], acc[r][c]);
      } else {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            if (c < DPXC) {
              acc[r][c] = __viaddmin_s32(x0[r], b0[c], acc[r][c]);
              acc[r][c] = __viaddmin_s32(x1[r], b1[c], acc[r][c]);
            } else {
              const int32_t s0 = x0[r] * one + b0[c];
              const int32_t s1 = x1[r] * one + b1[c];
              acc[r][c] = __vimin3_s32(acc[r][c], s0, s1);
            }
          }
      }
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int64_t i = i0 + (r >> 2) * 64 + ty * 4 + (r & 3);
    if (i >= M) continue;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int64_t j = j0 + (c >> 2) * 64 + tx * 4 + (c & 3);
      if (j >= N) continue;
      int32_t v = acc[r][c];
      if (accumulate) v = min(v, min(C[i * ldc + j], kInf32));
      C[i * ldc + j] = v;
    }
  }
}

template <int OUT, bool STATS, int DPXC, bool TMA, bool SK, int TN>
int launch_gemm_v(const uint32_t *XT, int64_t ldx, const uint32_t *BP, int64_t ldb, int64_t kpairs, void *C,
                  int64_t ldc, int64_t M, int64_t N, int64_t Mp, int64_t Np, const EpiArgs &epi,
                  cudaStream_t st, int nsplit, const PeerB &pb, const TmaOps *tma) {
  static bool attr_set[64] = {};
  const size_t smem = (size_t)kStages * kBK2 * (kTile + TN) * 4 + (TMA ? 1024 : 0);
  int dev = 0;
  RD_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    RD_CUDA_CHECK(cudaFuncSetAttribute(minplus_gemm_kernel<OUT, STATS, DPXC, TMA, SK, TN>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  const int nti = (int)(Mp / kTile), ntj = (int)(Np / TN);
  TmaOps t{};
  if (tma) t = *tma;
  // stream-K steps: sk_nfull whole-tile CTAs, then sk_nsk CTAs sharing the remaining tiles
  // tail-split steps: tail_nfull whole-tile CTAs, then tail_split CTAs per remaining tile
  const unsigned gx = SK ? (unsigned)(epi.sk_nfull + epi.sk_nsk)
                    : epi.tail_split > 1 ? (unsigned)(epi.tail_nfull + (nti * ntj - epi.tail_nfull) * epi.tail_split)
                                         : (unsigned)(nti * ntj);
  minplus_gemm_kernel<OUT, STATS, DPXC, TMA, SK, TN><<<dim3(gx, (unsigned)nsplit), kThreads, smem, st>>>(
      XT, ldx, BP, ldb, (int)kpairs, C, ldc, M, N, nti, ntj, 1u, epi, g_raster_group, pb, t);
  RD_CUDA_CHECK(cudaGetLastError());
  return RD_OK;
}

template <int DPXC>
int launch_gemm32_v(const int32_t *XT, int64_t ldx, const int32_t *BP, int64_t ldb, int64_t kp, int32_t *C,
                    int64_t ldc, int64_t M, int64_t N, int64_t Mp, int64_t Np, int accumulate, cudaStream_t st) {
  static bool attr_set[64] = {};
  int dev = 0;
  RD_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    RD_CUDA_CHECK(cudaFuncSetAttribute(minplus_gemm32_kernel<DPXC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kSmemBytes));
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  const int nti = (int)(Mp / kTile), ntj = (int)(Np / kTile);
  minplus_gemm32_kernel<DPXC><<<(unsigned)(nti * ntj), kThreads, kSmemBytes, st>>>(
      XT, ldx, BP, ldb, (int)kp, C, ldc, M, N, nti, ntj, 1, accumulate, g_raster_group);
  RD_CUDA_CHECK(cudaGetLastError());
  return RD_OK;
}


}  // namespace rd

// Explicit instantiation of one launcher: RD_INST_GEMM(OUT, STATS, DPXC, TMA)
#define RD_INST_GEMM(OUT, STATS, D, TMA, ...)                                                              \
  template int rd::launch_gemm_v<OUT, STATS, D, TMA, ##__VA_ARGS__>(const uint32_t *, int64_t, const uint32_t *, int64_t,  \
                                                     int64_t, void *, int64_t, int64_t, int64_t, int64_t,  \
                                                     int64_t, const rd::EpiArgs &, cudaStream_t, int,      \
                                                     const rd::PeerB &, const rd::TmaOps *);
// TN = 64 instances (PM output, cp.async): RD_INST_GEMM64_ALL(STATS)
#define RD_INST_GEMM64(STATS, D)                                                                           \
  template int rd::launch_gemm_v<rd::kOutPM, STATS, D, false, false, 64>(                                  \
      const uint32_t *, int64_t, const uint32_t *, int64_t, int64_t, void *, int64_t, int64_t, int64_t,     \
      int64_t, int64_t, const rd::EpiArgs &, cudaStream_t, int, const rd::PeerB &, const rd::TmaOps *);
#define RD_INST_GEMM64_ALL(STATS) \
  RD_INST_GEMM64(STATS, 0) RD_INST_GEMM64(STATS, 2) RD_INST_GEMM64(STATS, 3) RD_INST_GEMM64(STATS, 4) RD_INST_GEMM64(STATS, 8)
#define RD_INST_GEMM_ALL(OUT, STATS, TMA, ...)                                                               \
  RD_INST_GEMM(OUT, STATS, 0, TMA, ##__VA_ARGS__) RD_INST_GEMM(OUT, STATS, 2, TMA, ##__VA_ARGS__)             \
  RD_INST_GEMM(OUT, STATS, 3, TMA, ##__VA_ARGS__) RD_INST_GEMM(OUT, STATS, 4, TMA, ##__VA_ARGS__)             \
  RD_INST_GEMM(OUT, STATS, 8, TMA, ##__VA_ARGS__)
