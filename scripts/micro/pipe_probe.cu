// Which pipe issues HMNMX2 / HADD2 / VIMNMX3 / PRMT on sm_100a: one kernel per
// op, 8 independent chains; read with ncu --metrics sm__inst_executed_pipe_*.
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 h(uint32_t x) { return *reinterpret_cast<__half2*>(&x); }
template <int OP>
__global__ void k(uint32_t* out, uint32_t seed, int iters) {
    uint32_t r[8];
    for (int i = 0; i < 8; ++i) r[i] = seed * (threadIdx.x + i + 1);
    const uint32_t c = seed ^ 0x1234u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) r[i] = u(__hmax2(h(r[i]), h(r[(i + 3) & 7])));
            if (OP == 1) r[i] = u(__hadd2_sat(h(r[i]), h(c + i)));
            if (OP == 2) r[i] = __vimax3_u16x2(r[i], c, c + i);
            if (OP == 3) r[i] = __byte_perm(r[i], c, 0x4140 + i);
            if (OP == 4) r[i] = __viaddmax_s16x2(r[i], c, c + i);
            if (OP == 5) r[i] = u(__hmin2(h(r[i]), h(r[(i + 5) & 7])));
        }
    }
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s ^= r[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    uint32_t* d;
    cudaMalloc(&d, 148 * 8 * 1024 * 4);
    k<0><<<148 * 8, 1024>>>(d, 7, 2000);
    k<1><<<148 * 8, 1024>>>(d, 7, 2000);
    k<2><<<148 * 8, 1024>>>(d, 7, 2000);
    k<3><<<148 * 8, 1024>>>(d, 7, 2000);
    k<4><<<148 * 8, 1024>>>(d, 7, 2000);
    k<5><<<148 * 8, 1024>>>(d, 7, 2000);
    cudaDeviceSynchronize();
    printf("ok\n");
}
