// Explicit instances of the (min,+) GEMM launchers (rd_gemm_kernels.cuh); one unit per
// group so that the build compiles them in parallel.
#include "rd_gemm_kernels.cuh"

RD_INST_GEMM_ALL(rd::kOutPM, true, true)
