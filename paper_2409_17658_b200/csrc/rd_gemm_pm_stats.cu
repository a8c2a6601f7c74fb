// Explicit instances of the (min,+) GEMM launchers (rd_gemm_kernels.cuh); one unit per
// group so that the build compiles them in parallel.
#include "rd_gemm_kernels.cuh"

RD_INST_GEMM_ALL(rd::kOutPM, true, false)
RD_INST_GEMM(rd::kOutPM, true, 13, false)
RD_INST_GEMM(rd::kOutPM, true, 14, false)
RD_INST_GEMM(rd::kOutPM, false, 13, false)
RD_INST_GEMM(rd::kOutPM, false, 14, false)
RD_INST_GEMM(rd::kOutPM, false, 13, true)
RD_INST_GEMM(rd::kOutPM, false, 14, true)
RD_INST_GEMM(rd::kOutRow, false, 13, false)
RD_INST_GEMM(rd::kOutRow, false, 14, false)
