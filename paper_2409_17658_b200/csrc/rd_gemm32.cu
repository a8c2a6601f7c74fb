// Explicit instances of the 32-bit (min,+) GEMM launchers (rd_gemm_kernels.cuh).
#include "rd_gemm_kernels.cuh"

template int rd::launch_gemm32_v<0>(const int32_t *, int64_t, const int32_t *, int64_t, int64_t, int32_t *, int64_t,
                                        int64_t, int64_t, int64_t, int64_t, int, cudaStream_t);
template int rd::launch_gemm32_v<2>(const int32_t *, int64_t, const int32_t *, int64_t, int64_t, int32_t *, int64_t,
                                        int64_t, int64_t, int64_t, int64_t, int, cudaStream_t);
template int rd::launch_gemm32_v<3>(const int32_t *, int64_t, const int32_t *, int64_t, int64_t, int32_t *, int64_t,
                                        int64_t, int64_t, int64_t, int64_t, int, cudaStream_t);
template int rd::launch_gemm32_v<4>(const int32_t *, int64_t, const int32_t *, int64_t, int64_t, int32_t *, int64_t,
                                        int64_t, int64_t, int64_t, int64_t, int, cudaStream_t);
template int rd::launch_gemm32_v<8>(const int32_t *, int64_t, const int32_t *, int64_t, int64_t, int32_t *, int64_t,
                                        int64_t, int64_t, int64_t, int64_t, int, cudaStream_t);
