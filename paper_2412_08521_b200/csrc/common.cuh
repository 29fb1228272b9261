// common.cuh -- shared helpers for the EMS sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <functional>

#include "ems_b200.h"

namespace ems {

constexpr int kWarp = 32;

// Internal select mode (never a descriptor policy): rank caller-supplied pooled scores passed in
// the glo slot (partition_tokens, compressor.cpp:48-74) with the EMS caps.
constexpr int kPolicyPooled = 100;

// Device-side status word (first 16 bytes of the workspace).
struct DevStatus {
    int32_t code;  // first error recorded (atomicCAS from 0)
    int32_t unit;
    int32_t pad[2];
};

__device__ __forceinline__ void record_status(DevStatus* st, int code, int unit) {
    if (atomicCAS(&st->code, 0, code) == 0) st->unit = unit;
}

template <typename T>
struct Elem;
template <>
struct Elem<float> {
    static __device__ __forceinline__ float load(const float* p) { return *p; }
    static __device__ __forceinline__ float to_float(float x) { return x; }
    static __device__ __forceinline__ float from_float(float x) { return x; }
};
template <>
struct Elem<__nv_bfloat16> {
    static __device__ __forceinline__ float load(const __nv_bfloat16* p) {
        return __bfloat162float(*p);
    }
    static __device__ __forceinline__ float to_float(__nv_bfloat16 x) { return __bfloat162float(x); }
    static __device__ __forceinline__ __nv_bfloat16 from_float(float x) {
        return __float2bfloat16_rn(x);
    }
};

template <typename T>
__device__ __forceinline__ float ld(const T* p) {
    return Elem<T>::load(p);
}
template <typename T>
__device__ __forceinline__ void st(T* p, float x) {
    *p = Elem<T>::from_float(x);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Inclusive block-wide prefix sum of one int per thread (blockDim.x = 32 * nwarps <= 1024):
// warp shuffles + one pass over the warp totals.  sh: >= 32 ints of shared memory.
__device__ __forceinline__ int block_incl_scan(int x, int* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) sh[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int t = lane < nw ? sh[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < nw) sh[lane] = t;
    }
    __syncthreads();
    return x + (warp > 0 ? sh[warp - 1] : 0);
}

// Host-side helpers shared by the launchers.
struct Dims {
    int B, Hq, Hkv, G, L, d, units;
    int lwin_scores;   // min(l_win, L)
    int cap_c, cap_l, cap_lut, cap_tbm;
    size_t esize;      // bytes per element of the dtype
    int unit_base = 0; // absolute index of unit 0 (chunked host pipeline), for status reports
};

Dims make_dims(const ems_desc& d);

// The forward pass of one problem in head parts whose Q lands in pieces (the first unit group of
// ems_prefill_host): `before(p, s)` is enqueued ahead of part p's forward launch (the wait for
// that part's host-to-device copy and its RoPE); part p covers query heads [p G/n, (p+1) G/n) of
// every unit.  Paths that cannot split run every `before` first.
struct ScoreParts {
    int n = 0;
    std::function<cudaError_t(int part, cudaStream_t s)> before;
};

void set_error(const char* fmt, ...);

// One NVTX range per C-ABI call (header-only NVTX 3: a no-op unless a profiler is attached), so
// nsight / ncu timelines show which entry point launched which kernels.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
#define EMS_NVTX(name) ::ems::NvtxRange ems_nvtx_range_(name)

// Dynamic shared memory above 48 KB is a function attribute of the CURRENT DEVICE's context:
// set it once per (kernel, device), so one process can drive several GPUs (one host thread
// per device).  Thread-safe; returns the cudaFuncSetAttribute status.
cudaError_t smem_optin(const void* kernel, int bytes);
// Clusters of `cluster` CTAs of `kernel` (threads, dynamic smem) co-resident on the current
// device (persistent grids); cached per kernel and device, after smem_optin.
int active_clusters(const void* kernel, int threads, int smem_bytes, int cluster);

#define EMS_CUDA_CHECK(expr)                                                          \
    do {                                                                              \
        cudaError_t _e = (expr);                                                      \
        if (_e != cudaSuccess) {                                                      \
            ::ems::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,               \
                             cudaGetErrorString(_e));                                 \
            return EMS_CUDA_ERROR;                                                    \
        }                                                                             \
    } while (0)

#define EMS_LAUNCH_CHECK()                                                            \
    do {                                                                              \
        cudaError_t _e = cudaGetLastError();                                          \
        if (_e != cudaSuccess) {                                                      \
            ::ems::set_error("%s:%d launch: %s", __FILE__, __LINE__,                  \
                             cudaGetErrorString(_e));                                 \
            return EMS_CUDA_ERROR;                                                    \
        }                                                                             \
    } while (0)

// ---- thread-block clusters: distributed shared memory reads, cluster barrier, rank --------
__device__ __forceinline__ uint32_t dsm_addr(const void* p, int rank) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"((uint32_t)__cvta_generic_to_shared(p)),
                 "r"(rank));
    return a;  // shared::cluster address, read with ld.shared::cluster
}
__device__ __forceinline__ int ld_dsm_i32(const void* p, int rank) {
    int v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(dsm_addr(p, rank)) : "memory");
    return v;
}
__device__ __forceinline__ long long ld_dsm_i64(const void* p, int rank) {
    long long v;
    asm volatile("ld.shared::cluster.s64 %0, [%1];" : "=l"(v) : "r"(dsm_addr(p, rank)) : "memory");
    return v;
}
__device__ __forceinline__ float ld_dsm_f32(const void* p, int rank) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(dsm_addr(p, rank)) : "memory");
    return v;
}
__device__ __forceinline__ double ld_dsm_f64(const void* p, int rank) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(dsm_addr(p, rank)) : "memory");
    return v;
}
// remote stores into another CTA's shared memory (visible to it after the next cl_sync)
__device__ __forceinline__ void st_dsm_i32(void* p, int rank, int v) {
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(dsm_addr(p, rank)), "r"(v) : "memory");
}
__device__ __forceinline__ void st_dsm_i64(void* p, int rank, long long v) {
    asm volatile("st.shared::cluster.s64 [%0], %1;" ::"r"(dsm_addr(p, rank)), "l"(v) : "memory");
}
__device__ __forceinline__ void st_dsm_f64(void* p, int rank, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(dsm_addr(p, rank)), "d"(v) : "memory");
}
// all threads of every CTA of the cluster; release/acquire at cluster scope (shared and global)
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cl_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

}  // namespace ems
