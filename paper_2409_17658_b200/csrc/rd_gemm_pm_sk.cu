// Explicit instances of the stream-K (min,+) GEMM launchers (rd_gemm_kernels.cuh): PM output,
// fused stats for the whole-tile CTAs, partial tiles for the stream-K CTAs.
#include "rd_gemm_kernels.cuh"

RD_INST_GEMM_ALL(rd::kOutPM, true, false, true)
RD_INST_GEMM_ALL(rd::kOutPM, true, true, true)
