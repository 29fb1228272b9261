// colsum_tc.cu -- (P2) KV-stationary column sums of the causal softmax, the
// Global-Local score of EMS ("modifying the loop order").
//
//   glo_j = (1/G) sum_h sum_{i >= j} P^h_ij ,  loc_j = (1/G) sum_h sum_{i >= L-w} P^h_ij
//   P^h_ij = exp2(q_i.k_j * c - lse2^h_i)   (exactly normalised with P1's row LSE)
// Reference semantics: streaming_pass column scatter, proj/src/scoring.cpp:52-62;
// GQA mean per contract D2.
//
// The row normalisation rides in the MMA: P1 writes x_i = -lse2_i / c as three bf16 terms (qx),
// and every S^T tile gets one more K = 16 step, K' = [K, 1 ... 1] against Q' = [Q, x1 x2 x3 0 ...],
// so the accumulator holds S' = q.k + x and the epilogue is exp2(S' c): no LSE loads from shared
// memory next to the exponentials (measured -4.6 % P2 time; the extra step is 1/8 more MMA work in
// a pass bound by the exponentials).  The split of x carries it to ~1e-6 absolute; glo agrees
// with the reference to ~1e-6 at full size (tests/test_gpu_fullsize_ref.py).
//
// Any L: the last query / key tile is TMA zero fill past L; queries >= L are masked in the
// (always masked-path) last query tile and keys >= L are never stored.
//
// One CTA owns TWO 128-key tiles (J0 = 2*jp, J1 = J0 + 1) of one unit, both resident in smem,
// and streams every (query head h, query-tile PAIR (I, I+1), I >= J0) through a 2-stage TMA ring
// (one 256-row box per 64 d-columns, plus the pair's qx rows).  Each pair feeds two SS MMAs
// S'^T_w = K'_Jw [Q'_I; Q'_I+1]^T with N = 256 (keys on TMEM lanes; ~90 % of the tensor rate
// against ~60 % for N = 128: same time -- the pass is bound by the exponentials -- and 2.6 % less
// energy per step), TMEM buffer w holding key tile Jw.  Four column warpgroups: per item
// (pair, w) warpgroup q owns query columns [64 q, 64 q + 64) of the pair and thread m owns key
// Jw*128 + m, so the column sum over queries is an in-thread row sum (no atomics).  Interior
// items take a mask-free path where kPoly of every 8 exp2 pairs run as a degree-5 polynomial on
// the FMA pipe (ex2_poly2) and the rest on MUFU.  Per-item fp32 sums are accumulated in fp64 in
// item order and the four column quarters are combined in a fixed order -> deterministic.
#include "score_tc.cuh"

namespace ems {

namespace {

using namespace tc;
using namespace sc;

constexpr int kQStages = 2;              // query-tile PAIRS: 2 x 64 KB
constexpr int kBufs = 2;                 // TMEM: buffer w holds S^T of key tile J0 + w (256 query cols)
constexpr int kThreads = 640;            // w0 TMA, w1 MMA, w2-3 spare, w4-19 column sums
constexpr int kPairBytes = 2 * kTileBytes;   // 256 query rows x 128 d
constexpr int kQxBytes = 256 * 32;           // the pair's qx rows: 256 x 16 bf16 (SWIZZLE_32B)
constexpr int kStageBytes = kPairBytes + kQxBytes;
constexpr int kOnesBytes = 128 * 32;         // K's extra columns: 128 x 16 bf16 ones
constexpr size_t kSmem = 1024 + 2 * kTileBytes + kOnesBytes + kQStages * kStageBytes;
static_assert(2 * 2 * 4 * 128 * 8 <= kQStages * kStageBytes, "the final combine reuses the Q ring");

struct Bars {
    uint64_t k_full;
    uint64_t q_full[kQStages], q_empty[kQStages];
    uint64_t s_full[kBufs], s_empty[kBufs];
    uint32_t tmem_base;
};

// 64 query columns of the thread's key row, general path (causal mask + window).
__device__ __forceinline__ void cols_masked(const uint32_t (&r)[2][32], float c, int q0, int key,
                                            int loc_start, int L, float& sg, float& sl) {
    sg = 0.f;
    sl = 0.f;
#pragma unroll
    for (int cc = 0; cc < 2; ++cc)
#pragma unroll
        for (int x = 0; x < 32; ++x) {
            const int n = cc * 32 + x, qi = q0 + n;
            float p = ex2(__uint_as_float(r[cc][x]) * c);  // S' c = s c - lse2 (qx fold)
            if (qi < key || qi >= L) p = 0.f;  // query before key, or padding row past L: masked
            sg += p;
            if (qi >= loc_start) sl += p;
        }
}

// 64 query columns, interior tile: no masks.  c = log2(e)/sqrt(128) is a literal (the
// tensor-core path is d = 128 only); groups of 4 pairs are tree-summed before entering
// one of 4 independent accumulators, keeping the FADD dependency chains short.
constexpr float kC128 = 0.12751743f;
constexpr int kPoly = 2;  // exp2 pairs (of every 8) computed on the FMA pipe (ex2_poly2; 0-3 measured, 2 fastest)
__device__ __forceinline__ float cols_fast(const uint32_t (&r)[2][32]) {
    const float2 c2 = make_float2(kC128, kC128);
    float2 acc[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) acc[g] = make_float2(0.f, 0.f);
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
#pragma unroll
        for (int x = 0; x < 32; x += 8) {
            float2 p[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 arg = __fmul2_rn(
                    make_float2(__uint_as_float(r[cc][x + 2 * e]), __uint_as_float(r[cc][x + 2 * e + 1])), c2);
                p[e] = ((x / 2 + e) & 7) < kPoly ? ex2_poly2(arg) : make_float2(ex2(arg.x), ex2(arg.y));
            }
            const int g = (x / 8) & 3;
            acc[g] = __fadd2_rn(acc[g], __fadd2_rn(__fadd2_rn(p[0], p[1]), __fadd2_rn(p[2], p[3])));
        }
    }
    const float2 s = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
    return s.x + s.y;
}

// P2 with N = 256 MMAs: the CTA keeps its two key tiles resident and streams PAIRS of query tiles
// (one 256-row TMA box per 64 d-columns); every pair feeds two SS MMAs S^T_w = K_Jw [Q_I; Q_I+1]^T
// (M = 128, N = 256, ~90 % of the tensor rate against ~60 % for N = 128), buffer w of TMEM holding
// key tile J0 + w.  Per item (pair, w) all four column warpgroups work on key tile J0 + w, warpgroup
// q on query columns [64 q, 64 q + 64) of the pair.
__global__ void __launch_bounds__(kThreads, 1)
    colsum_tc_kernel(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tq,
                     const __grid_constant__ CUtensorMap tqx, const ColArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
    uint8_t* sk = sm;                                  // K_J0 | K_J1 (2 x 32 KB)
    uint8_t* sones = sk + 2 * kTileBytes;              // 128 x 16 bf16 ones (K's extra columns)
    uint8_t* sq = sones + kOnesBytes;                  // ring of (query pair, its qx rows)
    double* spart = reinterpret_cast<double*>(sq);     // [2 key tiles][2 g/l][4 q][128], after the loop
    __shared__ Bars bars;

    const int tid = threadIdx.x, warp = tid >> 5;
    const int per_jp = a.units * a.hsplit;
    const int jp = blockIdx.x / per_jp;
    const int unit = blockIdx.x % a.units;
    const int hg = (blockIdx.x % per_jp) / a.units;
    const int gh = a.G / a.hsplit;
    const int b = unit / a.Hkv, hk = unit % a.Hkv;
    const int J0 = 2 * jp;
    const bool has1 = J0 + 1 < a.nT;
    const int nw = has1 ? 2 : 1;
    const int span_p = (a.nT - J0 + 1) / 2;            // query-tile pairs (J0, J0+1), (J0+2, J0+3), ...
    const int n_pairs = gh * span_p;                   // pair p -> head hg*gh + p / span_p, tile J0 + 2 (p % span_p)

    // K' = [K, 1 ... 1]: every element of the extra 16 columns is one, so the extra K-step adds the
    // row sum of the query's qx entries (x1 + x2 + x3 = -lse2 / c) whatever the swizzle order
    for (int i = tid; i < kOnesBytes / 16; i += kThreads)
        reinterpret_cast<uint4*>(sones)[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    fence_proxy_async();  // generic-proxy stores -> visible to the tensor core (async proxy)
    if (warp == 0) {
        tmem_alloc<512>(&bars.tmem_base);
    } else if (warp == 1 && elect_one()) {
        mbar_init(&bars.k_full, 1);
        for (int s = 0; s < kQStages; ++s) {
            mbar_init(&bars.q_full[s], 1);
            mbar_init(&bars.q_empty[s], 1);
        }
        for (int s = 0; s < kBufs; ++s) {
            mbar_init(&bars.s_full[s], 1);
            mbar_init(&bars.s_empty[s], 16);   // one arrival per column warp
        }
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars.tmem_base;

    if (warp == 0) {
        // ------------------------------------------------------------- TMA producer
        if (elect_one()) {
            tma_prefetch(&tk);
            tma_prefetch(&tq);
            tma_prefetch(&tqx);
            mbar_expect_tx(&bars.k_full, (has1 ? 2 : 1) * kTileBytes);
            tma_load_3d(sk, &tk, &bars.k_full, 0, J0 * kTile, unit);
            tma_load_3d(sk + 16384, &tk, &bars.k_full, 64, J0 * kTile, unit);
            if (has1) {
                tma_load_3d(sk + kTileBytes, &tk, &bars.k_full, 0, (J0 + 1) * kTile, unit);
                tma_load_3d(sk + kTileBytes + 16384, &tk, &bars.k_full, 64, (J0 + 1) * kTile, unit);
            }
            for (int p = 0; p < n_pairs; ++p) {
                const int h = hg * gh + p / span_p, I = J0 + 2 * (p % span_p);
                const int plane = b * a.Hq + hk * a.G + h;
                const int s = p % kQStages;
                if (p >= kQStages) mbar_wait(&bars.q_empty[s], ((p / kQStages) - 1) & 1);
                uint8_t* dq = sq + s * kStageBytes;
                mbar_expect_tx(&bars.q_full[s], kStageBytes);
                tma_load_3d(dq, &tq, &bars.q_full[s], 0, I * kTile, plane);
                tma_load_3d(dq + kTileBytes, &tq, &bars.q_full[s], 64, I * kTile, plane);
                tma_load_3d(dq + kPairBytes, &tqx, &bars.q_full[s], 0, I * kTile, plane);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------- MMA issuer
        if (elect_one()) {
            const uint32_t id_s = idesc_bf16(128, 256, 0, 0);  // K (K-major) x [Q_I; Q_I+1]^T (K-major)
            const uint32_t ka[2] = {smem_u32(sk), smem_u32(sk + kTileBytes)};
            mbar_wait(&bars.k_full, 0);
            for (int p = 0; p < n_pairs; ++p) {
                const int s = p % kQStages;
                mbar_wait(&bars.q_full[s], (p / kQStages) & 1);
                const uint32_t qa = smem_u32(sq + s * kStageBytes);
                for (int w = 0; w < nw; ++w) {
                    if (p >= 1) mbar_wait(&bars.s_empty[w], (p - 1) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        mma_ss(tmem + w * 256, sdesc(kmajor_addr(ka[w], k), 16, 1024),
                               sdesc(qa + (k >> 2) * kTileBytes + (k & 3) * 32, 16, 1024), id_s, k > 0);
                    // the row normalisation: S' = S + ones x qx^T (one more K = 16 step)
                    mma_ss(tmem + w * 256, sdesc_sw32(smem_u32(sones)), sdesc_sw32(qa + kPairBytes), id_s, 1u);
                    mma_commit(&bars.s_full[w]);
                }
                mma_commit(&bars.q_empty[s]);
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------- column sums
        const int q = (warp - 4) >> 2;          // query columns [64 q, 64 q + 64) of each pair
        const int wi = warp & 3;
        const int mrow = wi * 32 + (tid & 31);  // key row within the key tile
        const int loc_start = a.L - a.lwin;
        double acc_g[2] = {0.0, 0.0}, acc_l[2] = {0.0, 0.0};
        const uint32_t s_full0 = smem_u32(&bars.s_full[0]), s_empty0 = smem_u32(&bars.s_empty[0]);
        const uint32_t sa0 = tmem + 64 * q + ((uint32_t)(wi * 32) << 16);
        for (int p = 0, I = J0; p < n_pairs; ++p) {
            const int q0 = I * kTile + 64 * q;  // first query of this warpgroup's columns
#pragma unroll
            for (int w = 0; w < 2; ++w) {
                if (w >= nw) break;
                mbar_wait_u(s_full0 + 8 * w, p & 1);
                tc_fence_after();
                const int key0 = (J0 + w) * kTile;  // first key of the tile; this thread: key0 + mrow
                if (q0 + 63 >= key0) {  // some column of the quarter is at or after some key
                    uint32_t r[2][32];
                    const uint32_t sa = sa0 + w * 256;
                    tmem_ld32(sa, r[0]);
                    tmem_ld32(sa + 32, r[1]);
                    tmem_ld_wait();
                    if (q0 > key0 + kTile - 1 && q0 + 63 < loc_start) {
                        acc_g[w] += (double)cols_fast(r);
                    } else {
                        float sg, sl;
                        cols_masked(r, a.c, q0, key0 + mrow, loc_start, a.L, sg, sl);
                        acc_g[w] += (double)sg;
                        acc_l[w] += (double)sl;
                    }
                }
                tc_fence_before();
                __syncwarp();
                if ((tid & 31) == 0) mbar_arrive_u(s_empty0 + 8 * w);
            }
            I += 2;
            if (I >= a.nT) I = J0;
        }
        // combine the four column quarters of each key tile in a fixed order
#pragma unroll
        for (int w = 0; w < 2; ++w) {
            spart[((w * 2 + 0) * 4 + q) * 128 + mrow] = acc_g[w];
            spart[((w * 2 + 1) * 4 + q) * 128 + mrow] = acc_l[w];
        }
        asm volatile("bar.sync 1, 512;" ::: "memory");
        if (q < nw) {  // warpgroup q writes key tile J0 + q
            const int w = q, key = (J0 + w) * kTile + mrow;
            const double* g = spart + (w * 2 + 0) * 4 * 128 + mrow;
            const double* l = spart + (w * 2 + 1) * 4 * 128 + mrow;
            const double sg = ((g[0] + g[128]) + g[256]) + g[384];
            const double sl = ((l[0] + l[128]) + l[256]) + l[384];
            if (key < a.L) {
                if (a.hsplit == 1) {
                    const size_t o = (size_t)unit * a.L + key;
                    a.glo[o] = (float)(sg / a.G);
                    a.loc[o] = (float)(sl / a.G);
                } else {
                    const size_t o = ((size_t)unit * a.hsplit + hg) * a.L + key;
                    a.part_g[o] = sg;
                    a.part_l[o] = sl;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

// glo/loc = (sum over head groups, in order) / G  -- deterministic
__global__ void colsum_reduce_kernel(const double* __restrict__ pg, const double* __restrict__ pl,
                                     float* __restrict__ glo, float* __restrict__ loc, int units, int L,
                                     int hsplit, int G) {
    const size_t n = (size_t)units * L;
    for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < n; x += (size_t)gridDim.x * blockDim.x) {
        const size_t u = x / L, l = x % L;
        double g = 0.0, c = 0.0;
        for (int h = 0; h < hsplit; ++h) {
            g += pg[(u * hsplit + h) * L + l];
            c += pl[(u * hsplit + h) * L + l];
        }
        glo[x] = (float)(g / G);
        loc[x] = (float)(c / G);
    }
}

}  // namespace

cudaError_t launch_colsum_tc(const ColArgs& a, const CUtensorMap& tk, const CUtensorMap& tq,
                             const CUtensorMap& tqx, cudaStream_t s) {
    cudaError_t e = smem_optin(reinterpret_cast<const void*>(colsum_tc_kernel), (int)kSmem);
    if (e != cudaSuccess) return e;
    const dim3 grid(((a.nT + 1) / 2) * a.units * a.hsplit);
    colsum_tc_kernel<<<grid, kThreads, kSmem, s>>>(tk, tq, tqx, a);
    e = cudaGetLastError();
    if (e != cudaSuccess || a.hsplit == 1) return e;
    colsum_reduce_kernel<<<4 * 148, 256, 0, s>>>(a.part_g, a.part_l, a.glo, a.loc, a.units, a.L, a.hsplit, a.G);
    return cudaGetLastError();
}

// Head split for load balance: the smallest power-of-two divisor of G that gives at least
// ~4 CTAs per SM (the heaviest key-tile pair otherwise dominates small unit counts).
int colsum_hsplit(int G, int nT, int units) {
    const int pairs = (nT + 1) / 2;
    int hs = 1;
    while (hs < G && G % (2 * hs) == 0 && (long long)pairs * units * hs < 4LL * 148) hs *= 2;
    return hs;
}

}  // namespace ems
