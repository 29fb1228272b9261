// merge_tc.cu -- kernel (3) on the tensor cores: redundancy of the to-be-merged
// tokens against the class centers + argmax destination, bf16, head_dim 128.
//
//   R[t][c] = clamp(cos(k_t, k_c)) * clamp(cos(v_t, v_c))      (analysis.cpp:51-69, D1)
//   dest[t] = argmax_c R[t][c] (ties -> lower column) if max >= tau else -1
//                                                             (compressor.cpp:76-95)
// 1. gather_kernel copies the TBM rows and the center rows of raw K/V into contiguous
//    zero-padded buffers (128-row multiples) and computes fp32 inverse norms
//    (0 for zero-norm rows -> similarity 0, cos_or_zero analysis.cpp:16-24).
// 2. assign_tc_kernel: one CTA per (unit, 128 TBM rows).  K_T/V_T tiles stay in smem;
//    center tiles stream through a 2-stage TMA ring; two SS MMAs per center tile
//    (K_T K_C^T and V_T V_C^T, M = N = 128, K = 128) land in a double-buffered TMEM
//    pair; two epilogue warpgroups alternate tiles, each thread owning one TBM row:
//    cosines = dot * inv_norm_row * inv_norm_col, clamp, product, running argmax in
//    increasing column order with strict '>' (reference tie rule).  The two
//    warpgroups' (best, column) are combined with the same rule -> deterministic.
#include <stdlib.h>

#include "score_tc.cuh"
#include "tmap.h"

namespace ems {

namespace {

using namespace tc;
using namespace sc;

// ------------------------------------------------------------------ gather
__global__ void __launch_bounds__(256) gather_kernel(
    const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v, int L,
    const int32_t* __restrict__ imp_idx, const int32_t* __restrict__ tbm_idx,
    const int32_t* __restrict__ counts, int cap_c, int cap_t, int pad_c, int pad_t,
    __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc, __nv_bfloat16* __restrict__ kt,
    __nv_bfloat16* __restrict__ vt, float* __restrict__ inv) {
    // inv layout per unit: [kc pad_c][vc pad_c][kt pad_t][vt pad_t]
    const int u = blockIdx.y;
    const int e = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int n_imp = counts[4 * u], n_tbm = counts[4 * u + 1];
    int idx = -1;
    __nv_bfloat16 *dk, *dv;
    float *ik, *iv;
    float* invu = inv + (size_t)u * 2 * (pad_c + pad_t);
    if (e < pad_c) {
        if (e < n_imp) idx = imp_idx[(size_t)u * cap_c + e];
        dk = kc + ((size_t)u * pad_c + e) * kD;
        dv = vc + ((size_t)u * pad_c + e) * kD;
        ik = invu + e;
        iv = invu + pad_c + e;
    } else if (e < pad_c + pad_t) {
        const int t = e - pad_c;
        if (t < n_tbm) idx = tbm_idx[(size_t)u * cap_t + t];
        dk = kt + ((size_t)u * pad_t + t) * kD;
        dv = vt + ((size_t)u * pad_t + t) * kD;
        ik = invu + 2 * pad_c + t;
        iv = invu + 2 * pad_c + pad_t + t;
    } else {
        return;
    }
    // 128 bf16 = 256 B per row: lane copies 8 bytes (4 elements) of K and of V
    uint2 a = make_uint2(0, 0), b = make_uint2(0, 0);
    if (idx >= 0) {
        a = reinterpret_cast<const uint2*>(k + ((size_t)u * L + idx) * kD)[lane];
        b = reinterpret_cast<const uint2*>(v + ((size_t)u * L + idx) * kD)[lane];
    }
    reinterpret_cast<uint2*>(dk)[lane] = a;
    reinterpret_cast<uint2*>(dv)[lane] = b;
    float sk = 0.f, sv = 0.f;
    const __nv_bfloat16* pa = reinterpret_cast<const __nv_bfloat16*>(&a);
    const __nv_bfloat16* pb = reinterpret_cast<const __nv_bfloat16*>(&b);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float x = __bfloat162float(pa[i]), y = __bfloat162float(pb[i]);
        sk = fmaf(x, x, sk);
        sv = fmaf(y, y, sv);
    }
    sk = warp_sum(sk);
    sv = warp_sum(sv);
    if (lane == 0) {
        *ik = sk > 0.f ? 1.f / sqrtf(sk) : 0.f;
        *iv = sv > 0.f ? 1.f / sqrtf(sv) : 0.f;
    }
}

// ------------------------------------------------------------------ similarity + argmax
constexpr int kStages = 2;
static_assert(kStages == 2, "stage s of tile c is TMEM buffer c & 1 (the producer waits on d_empty[s])");
constexpr int kThreads = 384;  // w0 TMA, w1 MMA, w4-7 epilogue A, w8-11 epilogue B
constexpr size_t kSmem = 1024 + 2 * kTileBytes + kStages * (2 * kTileBytes + 1024) + 2 * 128 * 8;

struct Bars {
    uint64_t t_full;
    uint64_t c_full[kStages], c_empty[kStages];
    uint64_t d_full[2], d_empty[2];
    uint32_t tmem_base;
};

struct AssignArgs {
    int units, pad_c, pad_t, cap_t, key_only;
    double tau;
    const int32_t* counts;
    const float* inv;
    int32_t* dest;
};

__global__ void __launch_bounds__(kThreads, 1)
    assign_tc_kernel(const __grid_constant__ CUtensorMap tkc, const __grid_constant__ CUtensorMap tvc,
                     const __grid_constant__ CUtensorMap tkt, const __grid_constant__ CUtensorMap tvt,
                     const AssignArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
    uint8_t* skt = sm;                          // K_T tile
    uint8_t* svt = skt + kTileBytes;            // V_T tile
    uint8_t* sring = svt + kTileBytes;          // stages x (K_C, V_C, inv_kc[128], inv_vc[128])
    float* sbest = reinterpret_cast<float*>(sring + kStages * (2 * kTileBytes + 1024));  // [128]
    int* sbcol = reinterpret_cast<int*>(sbest + 128);
    __shared__ Bars bars;

    const int tid = threadIdx.x, warp = tid >> 5;
    const int u = blockIdx.y, t0 = blockIdx.x * 128;
    const int n_imp = a.counts[4 * u], n_tbm = a.counts[4 * u + 1];
    if (t0 >= n_tbm || n_imp == 0) {
        // nothing to assign (rows past n_tbm are never read)
        if (n_imp == 0)
            for (int t = t0 + tid; t < min(n_tbm, t0 + 128); t += kThreads) a.dest[(size_t)u * a.cap_t + t] = -1;
        return;
    }
    const int n_ct = (n_imp + 127) / 128;
    const float* invu = a.inv + (size_t)u * 2 * (a.pad_c + a.pad_t);

    if (warp == 0) {
        tmem_alloc<512>(&bars.tmem_base);
    } else if (warp == 1 && elect_one()) {
        mbar_init(&bars.t_full, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&bars.c_full[s], 1);
            mbar_init(&bars.c_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars.d_full[s], 1);
            mbar_init(&bars.d_empty[s], 128);
        }
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars.tmem_base;

    if (warp == 0) {
        if (elect_one()) {
            mbar_expect_tx(&bars.t_full, 2 * kTileBytes);
            tma_load_3d(skt, &tkt, &bars.t_full, 0, t0, u);
            tma_load_3d(skt + 16384, &tkt, &bars.t_full, 64, t0, u);
            tma_load_3d(svt, &tvt, &bars.t_full, 0, t0, u);
            tma_load_3d(svt + 16384, &tvt, &bars.t_full, 64, t0, u);
            for (int c = 0; c < n_ct; ++c) {
                const int s = c % kStages;
                if (c >= kStages) {
                    mbar_wait(&bars.c_empty[s], ((c / kStages) - 1) & 1);
                    // the epilogue of tile c - 2 still reads this stage's column norms
                    mbar_wait(&bars.d_empty[s], ((c >> 1) - 1) & 1);
                }
                uint8_t* st = sring + s * (2 * kTileBytes + 1024);
                mbar_expect_tx(&bars.c_full[s], 2 * kTileBytes + 1024);
                tma_load_3d(st, &tkc, &bars.c_full[s], 0, c * 128, u);
                tma_load_3d(st + 16384, &tkc, &bars.c_full[s], 64, c * 128, u);
                tma_load_3d(st + kTileBytes, &tvc, &bars.c_full[s], 0, c * 128, u);
                tma_load_3d(st + kTileBytes + 16384, &tvc, &bars.c_full[s], 64, c * 128, u);
                bulk_load(st + 2 * kTileBytes, invu + c * 128, 512, &bars.c_full[s]);
                bulk_load(st + 2 * kTileBytes + 512, invu + a.pad_c + c * 128, 512, &bars.c_full[s]);
            }
        }
    } else if (warp == 1) {
        if (elect_one()) {
            const uint32_t id = idesc_bf16(128, 128, 0, 0);
            const uint32_t ka = smem_u32(skt), va = smem_u32(svt);
            mbar_wait(&bars.t_full, 0);
            for (int c = 0; c < n_ct; ++c) {
                const int s = c % kStages, b = c & 1;
                mbar_wait(&bars.c_full[s], (c / kStages) & 1);
                if (c >= 2) mbar_wait(&bars.d_empty[b], ((c >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t kc = smem_u32(sring + s * (2 * kTileBytes + 1024));
                const uint32_t vc = kc + kTileBytes;
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    mma_ss(tmem + 256 * b, sdesc(kmajor_addr(ka, k), 16, 1024),
                           sdesc(kmajor_addr(kc, k), 16, 1024), id, k > 0);
                if (!a.key_only) {
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        mma_ss(tmem + 256 * b + 128, sdesc(kmajor_addr(va, k), 16, 1024),
                               sdesc(kmajor_addr(vc, k), 16, 1024), id, k > 0);
                }
                mma_commit(&bars.d_full[b]);
                mma_commit(&bars.c_empty[s]);
            }
        }
    } else if (warp >= 4) {
        const int g = (warp - 4) >> 2;          // epilogue warpgroup: center tiles c = g, g+2, ...
        const int wi = warp & 3;
        const int row = wi * 32 + (tid & 31);
        const int t = t0 + row;
        const float ikt = invu[2 * a.pad_c + t], ivt = invu[2 * a.pad_c + a.pad_t + t];
        float best = -INFINITY;
        int best_c = 0;
        for (int c = g; c < n_ct; c += 2) {
            const int s = c % kStages, b = c & 1;
            mbar_wait(&bars.d_full[b], (c >> 1) & 1);
            tc_fence_after();
            const uint32_t ls = smem_u32(sring + s * (2 * kTileBytes + 1024) + 2 * kTileBytes);
            const uint32_t dk = tmem + 256 * b + ((uint32_t)(wi * 32) << 16);
#pragma unroll 1
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t rk[32], rv[32];
                tmem_ld32(dk + ch * 32, rk);
                if (!a.key_only) tmem_ld32(dk + 128 + ch * 32, rv);
                tmem_ld_wait();
#pragma unroll
                for (int x = 0; x < 32; ++x) {
                    const int col = c * 128 + ch * 32 + x;
                    const float ck = fminf(1.f, fmaxf(-1.f, __uint_as_float(rk[x]) * ikt *
                                                             lds32(ls + 4 * (ch * 32 + x))));
                    float r = ck;
                    if (!a.key_only)
                        r *= fminf(1.f, fmaxf(-1.f, __uint_as_float(rv[x]) * ivt *
                                                        lds32(ls + 512 + 4 * (ch * 32 + x))));
                    if (col < n_imp && r > best) best = r, best_c = col;  // strict: ties -> lower col
                }
            }
            tc_fence_before();
            mbar_arrive(&bars.d_empty[b]);
        }
        // combine the two warpgroups (ties -> lower column)
        if (g == 1) {
            sbest[row] = best;
            sbcol[row] = best_c;
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (g == 0 && t < n_tbm) {
            const float ob = sbest[row];
            const int oc = sbcol[row];
            if (ob > best || (ob == best && oc < best_c)) best = ob, best_c = oc;
            a.dest[(size_t)u * a.cap_t + t] = ((double)best >= a.tau) ? best_c : -1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

}  // namespace

size_t merge_tc_workspace(const Dims& dm) {
    const size_t pad_c = (dm.cap_c + 127) / 128 * 128, pad_t = (dm.cap_tbm + 127) / 128 * 128;
    return (size_t)dm.units * ((pad_c + pad_t) * kD * 2 * 2 + (pad_c + pad_t) * 2 * 4) + 1024;
}

bool merge_tc_supported(const Dims& dm, int dtype) {
    return dtype == EMS_BF16 && dm.d == kD && dm.cap_tbm > 0 && encode_fn() != nullptr;
}

cudaError_t launch_merge_tc(const Dims& dm, const void* k, const void* v, const ems_stage& sg,
                            double tau, int key_only, void* ws, cudaStream_t s) {
    const int pad_c = (dm.cap_c + 127) / 128 * 128, pad_t = (dm.cap_tbm + 127) / 128 * 128;
    const size_t U = dm.units;
    uint8_t* p = static_cast<uint8_t*>(ws);
    auto take = [&](size_t bytes) {
        uint8_t* r = p;
        p += (bytes + 255) / 256 * 256;
        return r;
    };
    auto* kc = reinterpret_cast<__nv_bfloat16*>(take(U * pad_c * kD * 2));
    auto* vc = reinterpret_cast<__nv_bfloat16*>(take(U * pad_c * kD * 2));
    auto* kt = reinterpret_cast<__nv_bfloat16*>(take(U * pad_t * kD * 2));
    auto* vt = reinterpret_cast<__nv_bfloat16*>(take(U * pad_t * kD * 2));
    auto* inv = reinterpret_cast<float*>(take(U * 2 * (pad_c + pad_t) * 4));
    dim3 gg((pad_c + pad_t + 7) / 8, dm.units);
    gather_kernel<<<gg, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(k),
                                     static_cast<const __nv_bfloat16*>(v), dm.L, sg.imp_idx, sg.tbm_idx,
                                     sg.part_counts, dm.cap_c, dm.cap_tbm, pad_c, pad_t, kc, vc, kt, vt,
                                     inv);
    CUtensorMap tkc, tvc, tkt, tvt;
    if (!make_tmap_bf16_3d(&tkc, kc, kD, pad_c, U, 128) || !make_tmap_bf16_3d(&tvc, vc, kD, pad_c, U, 128) ||
        !make_tmap_bf16_3d(&tkt, kt, kD, pad_t, U, 128) || !make_tmap_bf16_3d(&tvt, vt, kD, pad_t, U, 128))
        return cudaErrorInvalidValue;
    AssignArgs a;
    a.units = dm.units;
    a.pad_c = pad_c;
    a.pad_t = pad_t;
    a.cap_t = dm.cap_tbm;
    a.key_only = key_only;
    a.tau = tau;
    a.counts = sg.part_counts;
    a.inv = inv;
    a.dest = sg.dest;
    cudaError_t e = smem_optin(reinterpret_cast<const void*>(assign_tc_kernel), (int)kSmem);
    if (e != cudaSuccess) return e;
    dim3 ga(pad_t / 128, dm.units);
    assign_tc_kernel<<<ga, kThreads, kSmem, s>>>(tkc, tvc, tkt, tvt, a);
    return cudaGetLastError();
}

}  // namespace ems
