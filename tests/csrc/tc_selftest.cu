// tc_selftest.cu -- TEST ONLY: single-CTA checks of the tcgen05 / TMA / descriptor
// primitives in paper_2412_08521_b200/csrc/tc.cuh against torch matmuls
// (tests/test_gpu_tc_primitives.py).  Built into tests/_build/libems_selftest.so.
#include <cuda_runtime.h>

#include "tc.cuh"
#include "tmap.h"

using namespace ems;
using namespace ems::tc;

namespace {

// mode bit 0: B is MN-major ([K][N] in global) instead of K-major ([N][K]);
// mode bit 1: A is staged into TMEM by the threads (TS MMA) instead of smem (SS).
__global__ void __launch_bounds__(128) selftest_kernel(const __grid_constant__ CUtensorMap ta,
                                                       const __grid_constant__ CUtensorMap tb,
                                                       const __nv_bfloat16* A, float* D, int mode) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = sm;              // 32 KB: A as two 128x64 SW128 boxes
    uint8_t* sb = sm + 32768;      // 32 KB: B likewise
    __shared__ uint64_t bar_load, bar_mma;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    const bool b_mn = mode & 1, a_tmem = mode & 2;
    if (warp == 0) tmem_alloc<256>(&tmem_base);
    if (tid == 0) {
        mbar_init(&bar_load, 1);
        mbar_init(&bar_mma, 1);
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tmem_base;
    if (tid == 0) {
        mbar_expect_tx(&bar_load, 65536);
        tma_load_3d(sa, &ta, &bar_load, 0, 0, 0);
        tma_load_3d(sa + 16384, &ta, &bar_load, 64, 0, 0);
        tma_load_3d(sb, &tb, &bar_load, 0, 0, 0);
        tma_load_3d(sb + 16384, &tb, &bar_load, 64, 0, 0);
    }
    if (a_tmem) {  // thread m writes row m of A (bf16 pairs) into TMEM columns 128..191
        uint32_t r[32];
        for (int c = 0; c < 2; ++c) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const __nv_bfloat16* p = A + tid * 128 + c * 64 + 2 * j;
                r[j] = pack_bf16(__bfloat162float(p[0]), __bfloat162float(p[1]));
            }
            tmem_st32(tm + ((uint32_t)(warp * 32) << 16) + 128 + c * 32, r);
        }
        tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        mbar_wait(&bar_load, 0);
        tc_fence_after();
        const uint32_t idesc = idesc_bf16(128, 128, 0, b_mn ? 1 : 0);
        for (int k = 0; k < 8; ++k) {
            const uint32_t a_addr = smem_u32(sa) + (k >> 2) * 16384 + (k & 3) * 32;
            const uint64_t bd = b_mn ? sdesc(smem_u32(sb) + k * 2048, 16384, 1024)
                                     : sdesc(smem_u32(sb) + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
            if (a_tmem)
                mma_ts(tm, tm + 128 + k * 8, bd, idesc, k > 0);
            else
                mma_ss(tm, sdesc(a_addr, 16, 1024), bd, idesc, k > 0);
        }
        mma_commit(&bar_mma);
    }
    mbar_wait(&bar_mma, 0);
    tc_fence_after();
    for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32(tm + ((uint32_t)(warp * 32) << 16) + c * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) D[tid * 128 + c * 32 + j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<256>(tm);
}

}  // namespace

extern "C" __attribute__((visibility("default"))) int ems_tc_selftest(int mode, const void* A,
                                                                     const void* B, float* D) {
    CUtensorMap ta, tb;
    if (!make_tmap_bf16_3d(&ta, A, 128, 128, 1, 128)) return 1;
    if (!make_tmap_bf16_3d(&tb, B, 128, 128, 1, 128)) return 2;
    const int smem = 65536 + 1024;
    cudaFuncSetAttribute(selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    selftest_kernel<<<1, 128, smem>>>(ta, tb, (const __nv_bfloat16*)A, D, mode);
    if (cudaGetLastError() != cudaSuccess) return 3;
    if (cudaDeviceSynchronize() != cudaSuccess) return 4;
    return 0;
}
