// Explicit instances of the 128 x 64-tile (min,+) GEMM launchers (rd_gemm_kernels.cuh): PM
// output with and without the fused stats, cp.async mainloop, 3 CTAs per SM.
#include "rd_gemm_kernels.cuh"

RD_INST_GEMM64_ALL(true)
RD_INST_GEMM64_ALL(false)
