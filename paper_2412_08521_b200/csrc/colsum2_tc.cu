// colsum2_tc.cu -- (P2, CTA-pair variant) KV-stationary column sums on cta_group::2.
//
//   glo_j = (1/G) sum_h sum_{i >= j} P^h_ij,  loc_j = (1/G) sum_h sum_{i >= L-w} P^h_ij,
//   P^h_ij = exp2(q_i.k_j * c - lse2^h_i)   (proj/src/scoring.cpp:52-62, contract D2)
//
// A cluster of two CTAs owns key tiles J0 = 2*jp (rank 0) and J0 + 1 (rank 1).  Each
// item is one query head h and TWO query tiles (I, I+1): rank 0 loads Q_I, rank 1
// loads Q_{I+1}, and the leader issues one M = 256 (keys), N = 256 (queries) MMA
//   S^T = [K_J0; K_J0+1] [Q_I; Q_I+1]^T     (tcgen05.mma.cta_group::2, ~90% of peak
// per instruction vs ~60% for the N = 128 single-CTA MMA of colsum_tc.cu), so each
// CTA receives its 128 keys x 256 queries in TMEM.  Two epilogue warpgroups per CTA
// take the two query halves of every key row; TMEM is double-buffered (2 x 256 cols).
// Per-item fp32 sums accumulate in fp64 in a fixed order -> deterministic.
#include <stdlib.h>

#include "score_tc.cuh"
#include "tmap.h"

namespace ems {

namespace {

using namespace tc;
using namespace sc;

constexpr int kQStages = 3;
constexpr int kBufs = 2;
constexpr int kThreads = 384;  // w0 TMA, w1 MMA (leader), w4-7 query half 0, w8-11 query half 1
constexpr size_t kSmem = 1024 + kTileBytes + kQStages * kTileBytes + kBufs * 1024 + 2 * 128 * 8;

struct Bars {
    uint64_t k_full;                                   // leader: both K tiles landed
    uint64_t q_full[kQStages];                         // leader: both Q halves landed
    uint64_t q_empty[kQStages];                        // local (multicast commit)
    uint64_t s_full[kBufs];                            // local (multicast commit)
    uint64_t s_empty[kBufs];                           // leader: 512 epilogue arrivals
    uint64_t l_full[kBufs], l_empty[kBufs];            // local lse ring
    uint32_t tmem_base;
};

__device__ __forceinline__ void row_half(uint32_t sa, uint32_t lb, float c, int qtile, int ktile,
                                         int mrow, int L, int loc_start, bool fast, float& sg, float& sl) {
    sg = 0.f;
    sl = 0.f;
    if (fast) {
        const float2 c2 = make_float2(c, c);
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
            uint32_t r[2][32];
            tmem_ld32(sa + h2 * 64, r[0]);
            tmem_ld32(sa + h2 * 64 + 32, r[1]);
            tmem_ld_wait();
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const uint32_t lc = lb + (2 * h2 + cc) * 128;
                float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll
                for (int x = 0; x < 32; x += 4) {
                    const float4 lv = lds128(lc + 4 * x);
                    const float2 a0 = __ffma2_rn(
                        make_float2(__uint_as_float(r[cc][x]), __uint_as_float(r[cc][x + 1])), c2,
                        make_float2(lv.x, lv.y));
                    const float2 a1 = __ffma2_rn(
                        make_float2(__uint_as_float(r[cc][x + 2]), __uint_as_float(r[cc][x + 3])), c2,
                        make_float2(lv.z, lv.w));
                    // 3 of every 8 pairs through the FMA-pipe polynomial, the rest on MUFU
                    const float2 p0 = ((x / 2) & 7) < 3 ? ex2_poly2(a0) : make_float2(ex2(a0.x), ex2(a0.y));
                    const float2 p1 = ((x / 2 + 1) & 7) < 3 ? ex2_poly2(a1) : make_float2(ex2(a1.x), ex2(a1.y));
                    s0 = __fadd2_rn(s0, p0);
                    s1 = __fadd2_rn(s1, p1);
                }
                acc = __fadd2_rn(acc, __fadd2_rn(s0, s1));
            }
        }
        sg = acc.x + acc.y;
        return;
    }
    const int key = ktile * kTile + mrow;
#pragma unroll 1
    for (int h2 = 0; h2 < 2; ++h2) {
        uint32_t r[2][32];
        tmem_ld32(sa + h2 * 64, r[0]);
        tmem_ld32(sa + h2 * 64 + 32, r[1]);
        tmem_ld_wait();
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            const int c0 = (2 * h2 + cc) * 32;
#pragma unroll
            for (int x = 0; x < 32; ++x) {
                const int qi = qtile * kTile + c0 + x;
                float p = ex2(fmaf(__uint_as_float(r[cc][x]), c, lds32(lb + 4 * (c0 + x))));
                if (qi < key || qi >= L) p = 0.f;  // causal mask / past the prompt (TMA zero rows)
                sg += p;
                if (qi >= loc_start) sl += p;
            }
        }
    }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    colsum2_kernel(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tq,
                   const ColArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
    uint8_t* sk = sm;                                   // this CTA's key tile
    uint8_t* sq = sk + kTileBytes;                      // Q ring (this CTA's query half)
    float* slse = reinterpret_cast<float*>(sq + kQStages * kTileBytes);  // [kBufs][256]
    double* spart = reinterpret_cast<double*>(slse + kBufs * 256);       // [2][128]
    __shared__ Bars bars;

    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t rank = cluster_ctarank();
    const int pair = blockIdx.x >> 1;
    const int jp = pair / a.units, unit = pair % a.units;   // heaviest key tiles first
    const int b = unit / a.Hkv, hk = unit % a.Hkv;
    const int J0 = 2 * jp;
    const int Jr = J0 + (int)rank;                           // this CTA's key tile
    const int span = a.nT - J0;                              // query tiles J0 .. nT-1
    const int n_qp = (span + 1) / 2;                         // query-tile pairs per head
    const int n_items = a.G * n_qp;                          // item i: head i / n_qp, I = J0 + 2 (i % n_qp)

    if (warp == 0) {
        tmem_alloc_2sm<512>(&bars.tmem_base);
    } else if (warp == 1 && elect_one()) {
        mbar_init(&bars.k_full, 1);
        for (int s = 0; s < kQStages; ++s) {
            mbar_init(&bars.q_full[s], 1);
            mbar_init(&bars.q_empty[s], 1);
        }
        for (int s = 0; s < kBufs; ++s) {
            mbar_init(&bars.s_full[s], 1);
            mbar_init(&bars.s_empty[s], 16);   // 8 epilogue warps x 2 CTAs
            mbar_init(&bars.l_full[s], 1);
            mbar_init(&bars.l_empty[s], 8);
        }
        fence_barrier_init();
    }
    tc_fence_before();
    cluster_sync();  // barriers of both CTAs initialised before any remote arrive / TMA
    tc_fence_after();
    const uint32_t tmem = bars.tmem_base;

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA (both CTAs)
        if (elect_one()) {
            tma_prefetch(&tk);
            tma_prefetch(&tq);
            if (rank == 0) mbar_expect_tx(&bars.k_full, 2 * kTileBytes);
            tma_load_3d_2sm(sk, &tk, &bars.k_full, 0, Jr * kTile, unit);
            tma_load_3d_2sm(sk + 16384, &tk, &bars.k_full, 64, Jr * kTile, unit);
            for (int i = 0; i < n_items; ++i) {
                const int h = i / n_qp, I = J0 + 2 * (i % n_qp);
                const int plane = b * a.Hq + hk * a.G + h;
                const int s = i % kQStages, bb = i % kBufs;
                if (i >= kQStages) mbar_wait(&bars.q_empty[s], ((i / kQStages) - 1) & 1);
                if (rank == 0) mbar_expect_tx(&bars.q_full[s], 2 * kTileBytes);
                uint8_t* dq = sq + s * kTileBytes;
                const int qt = I + (int)rank;  // rank 1 supplies the second query tile (OOB rows -> 0)
                tma_load_3d_2sm(dq, &tq, &bars.q_full[s], 0, qt * kTile, plane);
                tma_load_3d_2sm(dq + 16384, &tq, &bars.q_full[s], 64, qt * kTile, plane);
                if (i >= kBufs) mbar_wait(&bars.l_empty[bb], ((i / kBufs) - 1) & 1);
                const int nl = (I + 1 < a.nT) ? 2 : 1;
                mbar_expect_tx(&bars.l_full[bb], nl * 512);
                bulk_load(slse + bb * 256, a.nlse2 + (size_t)plane * a.L + (size_t)I * kTile, nl * 512,
                          &bars.l_full[bb]);
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA (leader only)
        if (rank == 0 && elect_one()) {
            const uint32_t id = idesc_bf16(256, 256, 0, 0);
            const uint32_t ka = smem_u32(sk);
            mbar_wait(&bars.k_full, 0);
            for (int i = 0; i < n_items; ++i) {
                const int s = i % kQStages, bb = i % kBufs;
                mbar_wait(&bars.q_full[s], (i / kQStages) & 1);
                if (i >= kBufs) mbar_wait(&bars.s_empty[bb], ((i / kBufs) - 1) & 1);
                tc_fence_after();
                const uint32_t qa = smem_u32(sq + s * kTileBytes);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    mma_ss_2sm(tmem + bb * 256, sdesc(kmajor_addr(ka, k), 16, 1024),
                               sdesc(kmajor_addr(qa, k), 16, 1024), id, k > 0);
                mma_commit_2sm(&bars.s_full[bb], 0x3);
                mma_commit_2sm(&bars.q_empty[s], 0x3);
            }
        }
    } else if (warp >= 4) {
        // ---------------------------------------------------------------- column sums
        const int hq = (warp - 4) >> 2;          // query half: tile I + hq
        const int wi = warp & 3;
        const int mrow = wi * 32 + (tid & 31);
        const int loc_start = a.L - a.lwin;
        const int last_interior = loc_start / kTile - 1;
        const uint32_t s_empty_leader = mapa(smem_u32(&bars.s_empty[0]), 0);
        double acc_g = 0.0, acc_l = 0.0;
        for (int i = 0; i < n_items; ++i) {
            const int I = J0 + 2 * (i % n_qp);
            const int qt = I + hq;
            const int bb = i % kBufs;
            const uint32_t ph = (i / kBufs) & 1;
            mbar_wait(&bars.l_full[bb], ph);
            mbar_wait(&bars.s_full[bb], ph);
            tc_fence_after();
            if (qt >= Jr && qt < a.nT) {
                const uint32_t sa = tmem + bb * 256 + 128 * hq + ((uint32_t)(wi * 32) << 16);
                const uint32_t lb = smem_u32(slse + bb * 256 + 128 * hq);
                const bool fast = qt > Jr && qt <= last_interior;
                float sg, sl;
                row_half(sa, lb, a.c, qt, Jr, mrow, a.L, loc_start, fast, sg, sl);
                acc_g += (double)sg;
                acc_l += (double)sl;
            }
            tc_fence_before();
            __syncwarp();
            if ((tid & 31) == 0) {  // one (cluster-scope, fenced) arrival per warp
                mbar_arrive_cluster(s_empty_leader + bb * 8);
                mbar_arrive(&bars.l_empty[bb]);
            }
        }
        if (hq == 1) {
            spart[mrow] = acc_g;
            spart[128 + mrow] = acc_l;
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (hq == 0 && Jr < a.nT) {
            const size_t o = (size_t)unit * a.L + (size_t)Jr * kTile + mrow;
            a.glo[o] = (float)((acc_g + spart[mrow]) / a.G);
            a.loc[o] = (float)((acc_l + spart[128 + mrow]) / a.G);
        }
    }
    tc_fence_before();
    cluster_sync();  // the peer's TMEM / barriers stay alive until the leader is done
    if (warp == 0) tmem_dealloc_2sm<512>(tmem);
}

}  // namespace

cudaError_t launch_colsum2_tc(const ColArgs& a, const CUtensorMap& tk, const CUtensorMap& tq,
                              cudaStream_t s) {
    static const bool attr = [] {  // once per process, thread-safe (magic static)
        cudaFuncSetAttribute(colsum2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
        return true;
    }();
    (void)attr;
    const dim3 grid(2 * ((a.nT + 1) / 2) * a.units);
    colsum2_kernel<<<grid, kThreads, kSmem, s>>>(tk, tq, a);
    return cudaGetLastError();
}

}  // namespace ems
