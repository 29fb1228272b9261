// fwd2_tc.cu -- (P1) causal FlashAttention forward on CTA pairs (cta_group::2) with 256-key
// tiles: O, row LSE.  Reference semantics: streaming_pass, proj/src/scoring.cpp:20-64, for any
// prompt length L (the reference accepts any n) and any GQA group size G.
//
// Work item: two 128-row (query head, query tile) items of one unit, one per CTA of the pair.  A
// unit's G * ceil(L/128) items are walked heaviest tile first, heads inner, and paired
// consecutively (the same query tile of two heads when G is even; tiles t, t-1 of one head when
// G == 1); an odd item count gets a dummy partner that recomputes rank 0's item and stores
// nothing.  Rows >= L of the last query tile and keys >= L of the last key tile arrive as TMA
// zero fill; the causal mask (key > row) removes every key >= L from every real row, and no row
// >= L is stored.
//
// Persistent: one cluster per SM pair (as many as are co-resident) runs pairs until the launch's
// list is exhausted -- its first pair by cluster index, every later one from an atomic counter,
// published by the leader's TMA thread to every role of both CTAs through a 4-deep shared-memory
// ring (st.shared::cluster + a cluster-scope release arrive).  The hardware would list-schedule
// one cluster per pair the same way; keeping the CTAs resident removes the per-pair launch,
// TMEM allocation and pipeline fill (measured: 3.9 us to the first S and 1.8 us of teardown and
// relaunch gap per pair, 6 % of config 3 and 29 % at L = 4096), since the next pair's Q (double
// buffered) and first K/V tiles land while this pair computes and its first S runs under this
// pair's epilogue.  |q_row| for the logit bound is read from the Q tile in shared memory.
//
// The leader issues, per 256-key tile j of a pair,
//   S_j  = Q K_j^T        tcgen05.mma.cta_group::2, M = 256, N = 256, K = 128 (SS): each CTA
//                          supplies its 128 query rows (A) and one 128-key half of K_j (B)
//   O   += P_j V_j        M = 256, N = 128, K = 256 (TS: P from TMEM): each CTA supplies its
//                          P rows and a 64-column half of V_j (B, MN-major)
// (~92% / ~69% of the tensor rate).  TMEM per CTA: S [0,256) | P (bf16) [256,384) | O [384,512):
// P has its own columns, so S_{j+1} is issued as soon as both CTAs have read S_j into registers
// and runs under the softmax of tile j; PV_j follows in two K-halves, each issued as soon as its
// half of P_j is stored.  Softmax: four warpgroups per CTA, thread = (row, 32 keys of each
// 128-key half); row maxima exchanged through shared memory; lazily updated reference max (O
// rescaled only when a row max grows by > 8 in log2 units).  The normalised O tile is staged in
// the pair's (then idle) Q buffer and written by two bulk tensor stores (per-thread 16-byte row
// stores took 1.7 us per pair).  Warp roles: warps 0-15 softmax, 16 TMA + scheduler, 17 MMA,
// 18 O stores; setmaxnreg moves registers from the control warpgroup (16-19) to the softmax
// warpgroups (the launch allows 96 per thread: 5 warps share an SM sub-partition).
#include <cuda.h>
#include <stddef.h>
#include <stdlib.h>

#include "score_tc.cuh"

namespace ems {

namespace {

using namespace tc;
using namespace sc;

constexpr float kRescale2 = 8.0f;
// A tile whose logits provably stay below m_ref + kSkip (|q.k| <= |q| max|k|) needs neither its
// row max nor the max exchange: its p = 2^(s c - m_ref) <= 2^kSkip cannot overflow fp32/bf16.
constexpr float kSkip = 64.0f;
constexpr int kT2 = 640;  // w0-15 softmax (warpgroup q), w16 TMA + scheduler, w17 MMA (leader), w18 O stores
constexpr int kWTma = 16, kWMma = 17;
constexpr int kRegSoftmax = 104, kRegControl = 64;  // setmaxnreg per warpgroup (launch: 96)
constexpr int kStages2 = 2;
constexpr int kRing = 4;  // scheduled pairs in flight (leader -> every role of both CTAs)
// Q double buffer 2 x 32 KB | K stages (this CTA's 128-key half) | V stages (256 keys x this
// CTA's 64 d cols) | max/sum exchange
constexpr size_t kSmem2 = 1024 + 2 * kTileBytes + 2 * kStages2 * kTileBytes + 2 * 4 * 128 * 4;
constexpr int kMaxT2 = 4096;  // 256-key tiles per sequence (L <= 1048576)

struct Fwd2Args {
    int L, Lp, Hq, Hkv, G, nT, units;  // Lp = nT * 128: row stride of qx
    int h0, Gs;                        // this launch's query heads of every unit: h0 .. h0 + Gs - 1
    float c;
    __nv_bfloat16* out;  // [planes][L][128] (may be null)
    __nv_bfloat16* qx;   // [planes][Lp][16] -lse2/c as three bf16 terms (P2's extra K columns)
    float* lse_nat;      // [planes][L] natural-log LSE (may be null)
    const float* kmax;  // [units][nT2] max ||k|| over each 256-key tile (Cauchy-Schwarz bound)
    int nT2;
    int pairs;               // work items (CTA-pair items) of the launch
    int* next;               // dynamic scheduler: pairs handed out beyond the first wave (zeroed)
};

struct Bars2 {
    uint64_t q_full[2], q_empty[2];                 // leader (both halves) / local (multicast commit)
    uint64_t k_full[kStages2], v_full[kStages2];    // leader: both halves landed
    uint64_t k_empty[kStages2], v_empty[kStages2];  // local (multicast commit)
    uint64_t s_full, o_full;                        // local (multicast commit)
    uint64_t s_free, p_full, p_full_hi;             // leader: 32 warp arrivals (16 per CTA)
    uint64_t o_staged[2];                           // local: 16 softmax warps staged O (pair parity)
    uint64_t item_full[kRing];                      // local: the leader published the slot
    uint64_t item_empty[kRing];                     // leader: every consumer of both CTAs read it
    int item[kRing];
    uint32_t tmem_base;
};
// consumers of a scheduled pair: per CTA 16 softmax warps and the O store thread; the leader's
// MMA thread and the partner's TMA thread
constexpr int kItemConsumers = 2 * 17 + 2;
constexpr int kWStore = 18;  // O store thread (TMA bulk tensor stores from the staged tile)

struct Item {
    int plane, tile, unit, jmax;
    bool real;
};

// Unit by unit; within a unit item k = (tile nT-1 - k/G, head k%G), pairs (2p, 2p+1).
__device__ __forceinline__ Item pair_item(const Fwd2Args& a, int pair, int rank) {
    Item it;
    const int items = a.Gs * a.nT, per_unit = (items + 1) / 2;
    it.unit = pair / per_unit;
    const int k0 = 2 * (pair % per_unit);
    int k = k0 + rank;
    it.real = k < items;
    if (!it.real) k = k0;  // dummy partner: rank 0's item again, nothing stored
    it.tile = a.nT - 1 - k / a.Gs;
    const int b = it.unit / a.Hkv, hk = it.unit % a.Hkv;
    it.plane = b * a.Hq + hk * a.G + a.h0 + k % a.Gs;
    // 256-key tiles 0 .. jmax cover every key <= the last query row of both CTAs (rank 0's
    // item has the larger or equal tile)
    it.jmax = (a.nT - 1 - k0 / a.Gs) / 2;
    return it;
}

// Consumer side of the pair ring: wait for slot n, read it, release it to the leader (when
// `release`: one arrival per consuming warp or thread).
__device__ __forceinline__ int take_pair(Bars2& bars, int n, bool release) {
    const int s = n % kRing;
    mbar_wait_acq_cluster(smem_u32(&bars.item_full[s]), (n / kRing) & 1);
    const int idx = *reinterpret_cast<volatile int*>(&bars.item[s]);
    __syncwarp(__activemask());
    if (release) mbar_arrive_cluster(mapa(smem_u32(&bars.item_empty[s]), 0));
    return idx;
}

// Persistent cluster of two CTAs (see the file comment).  Per pair the MMA order is S_0, then
// S_{j+1} ahead of PV_j, and after the pair's last PV the next pair's S_0, which runs under this
// pair's epilogue.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kT2, 1)
    fwd2_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                   const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap to,
                   const Fwd2Args a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sq = sm;                                   // 2 x 32 KB: this CTA's 128 query rows
    uint8_t* sk = sq + 2 * kTileBytes;                  // stages x 32 KB: 128 keys x 128 d
    uint8_t* sv = sk + kStages2 * kTileBytes;           // stages x 32 KB: 256 keys x 64 d
    float* xch = reinterpret_cast<float*>(sv + kStages2 * kTileBytes);  // [2 buf][4 quarters][128]
    __shared__ Bars2 bars;

    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t rank = cluster_ctarank();

    if (warp == kWTma) {
        tmem_alloc_2sm<512>(&bars.tmem_base);
    } else if (warp == kWMma && elect_one()) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&bars.q_full[b], 1);
            // the pair's last S (MMA commit) + its O staged in this buffer stored (store thread)
            mbar_init(&bars.q_empty[b], 2);
            mbar_init(&bars.o_staged[b], 16);
        }
        for (int s = 0; s < kStages2; ++s) {
            mbar_init(&bars.k_full[s], 1);
            mbar_init(&bars.v_full[s], 1);
            mbar_init(&bars.k_empty[s], 1);
            mbar_init(&bars.v_empty[s], 1);
        }
        mbar_init(&bars.s_full, 1);
        mbar_init(&bars.o_full, 1);
        mbar_init(&bars.s_free, 32);
        mbar_init(&bars.p_full, 32);
        mbar_init(&bars.p_full_hi, 32);
        for (int s = 0; s < kRing; ++s) {
            mbar_init(&bars.item_full[s], 1);
            mbar_init(&bars.item_empty[s], kItemConsumers);
        }
        fence_barrier_init();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = bars.tmem_base;
    const uint32_t tS = tmem, tP = tmem + 256, tO = tmem + 384;

    // every role ends with the same teardown (each branch keeps its own register budget)
    auto teardown = [&]() {
        tc_fence_before();
        cluster_sync();
        if (warp == kWTma) tmem_dealloc_2sm<512>(tmem);
    };
    if (warp >= 16) {
        reg_dealloc<kRegControl>();  // the control warpgroup hands its registers to the softmax warpgroups
        if (warp == kWTma) {
            // ---------------------------------------------------------------- scheduler + TMA
            if (elect_one()) {
                tma_prefetch(&tq);
                tma_prefetch(&tk);
                tma_prefetch(&tv);
                int g = 0;  // 256-key tiles loaded so far (ring position across pairs)
                int ahead = 0;
                if (rank == 0) ahead = (int)(gridDim.x >> 1) + atomicAdd(a.next, 1);
                for (int n = 0;; ++n) {
                    int idx;
                    if (rank == 0) {  // publish pair n to both CTAs
                        const int s = n % kRing;
                        if (n >= kRing) mbar_wait(&bars.item_empty[s], ((n / kRing) - 1) & 1);
                        idx = n == 0 ? (int)(blockIdx.x >> 1) : ahead;
                        if (n > 0 && idx < a.pairs) ahead = (int)(gridDim.x >> 1) + atomicAdd(a.next, 1);
                        bars.item[s] = idx;
                        st_cluster_s32(mapa(smem_u32(&bars.item[s]), 1), idx);
                        mbar_arrive(&bars.item_full[s]);
                        mbar_arrive_release_cluster(mapa(smem_u32(&bars.item_full[s]), 1));
                    } else {
                        idx = take_pair(bars, n, true);
                    }
                    if (idx >= a.pairs) break;
                    const Item it = pair_item(a, idx, (int)rank);
                    const int qb = n & 1;
                    if (n >= 2) mbar_wait(&bars.q_empty[qb], ((n >> 1) - 1) & 1);
                    if (rank == 0) mbar_expect_tx(&bars.q_full[qb], 2 * kTileBytes);
                    uint8_t* dq = sq + qb * kTileBytes;
                    tma_load_3d_2sm(dq, &tq, &bars.q_full[qb], 0, it.tile * kTile, it.plane);
                    tma_load_3d_2sm(dq + 16384, &tq, &bars.q_full[qb], 64, it.tile * kTile, it.plane);
                    for (int j = 0; j <= it.jmax; ++j, ++g) {
                        const int s = g % kStages2;
                        const uint32_t ph = ((g / kStages2) - 1) & 1;
                        if (g >= kStages2) mbar_wait(&bars.k_empty[s], ph);
                        if (rank == 0) mbar_expect_tx(&bars.k_full[s], 2 * kTileBytes);
                        uint8_t* dk = sk + s * kTileBytes;
                        const int krow = 2 * j * kTile + (int)rank * kTile;  // this CTA's 128-key half
                        tma_load_3d_2sm(dk, &tk, &bars.k_full[s], 0, krow, it.unit);
                        tma_load_3d_2sm(dk + 16384, &tk, &bars.k_full[s], 64, krow, it.unit);
                        if (g >= kStages2) mbar_wait(&bars.v_empty[s], ph);
                        if (rank == 0) mbar_expect_tx(&bars.v_full[s], 2 * kTileBytes);
                        uint8_t* dv = sv + s * kTileBytes;  // keys 256j .. +255, d cols 64 rank .. +63
                        tma_load_3d_2sm(dv, &tv, &bars.v_full[s], 64 * (int)rank, 2 * j * kTile, it.unit);
                        tma_load_3d_2sm(dv + 16384, &tv, &bars.v_full[s], 64 * (int)rank, 2 * j * kTile + kTile,
                                        it.unit);
                    }
                }
            }
        } else if (warp == kWMma) {
            // ---------------------------------------------------------------- MMA (leader only)
            if (rank == 0 && elect_one()) {
                const uint32_t id_s = idesc_bf16(256, 256, 0, 0);  // Q (K-major) x K^T (K-major)
                const uint32_t id_o = idesc_bf16(256, 128, 0, 1);  // P (TMEM) x V (MN-major)
                // S of 256-key tile g from Q buffer qb; the pair's last S releases its Q buffer
                auto issue_s = [&](int g, int qb, bool last) {
                    // the K-steps' descriptors differ only in the start address (byte offset >> 4)
                    const uint64_t dq = sdesc(smem_u32(sq + qb * kTileBytes), 16, 1024);
                    const uint64_t dk = sdesc(smem_u32(sk + (g % kStages2) * kTileBytes), 16, 1024);
    #pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint64_t o = (uint64_t)(((k >> 2) << 10) + ((k & 3) << 1));  // kmajor_addr(.., k)
                        mma_ss_2sm(tS, dq + o, dk + o, id_s, k > 0);
                    }
                    mma_commit_2sm(&bars.s_full, 0x3);
                    mma_commit_2sm(&bars.k_empty[g % kStages2], 0x3);
                    if (last) mma_commit_2sm(&bars.q_empty[qb], 0x3);
                };
                int idx = take_pair(bars, 0, true);
                if (idx < a.pairs) {
                    Item it = pair_item(a, idx, 0);
                    mbar_wait(&bars.q_full[0], 0);
                    mbar_wait(&bars.k_full[0], 0);
                    tc_fence_after();
                    issue_s(0, 0, it.jmax == 0);
                    int g = 0;
                    for (int n = 0;; ++n) {
                        int nidx = a.pairs;
                        Item nit = it;
                        for (int j = 0; j <= it.jmax; ++j, ++g) {
                            // the next S of this pair (tile j+1) goes ahead of PV_g: it runs under the
                            // softmax of tile g
                            if (j < it.jmax) {
                                mbar_wait(&bars.s_free, g & 1);  // both CTAs hold S_g in registers
                                mbar_wait(&bars.k_full[(g + 1) % kStages2], ((g + 1) / kStages2) & 1);
                                tc_fence_after();
                                issue_s(g + 1, n & 1, j + 1 == it.jmax);
                            }
                            // PV_g in two K-halves: keys [0, 128) as soon as the softmax warps stored
                            // that half of P_g, keys [128, 256) after the other half.  Tile 0 of a pair
                            // overwrites O: its P arrives only after every softmax warp read the
                            // previous pair's O in its epilogue.
                            mbar_wait(&bars.p_full, g & 1);
                            mbar_wait(&bars.v_full[g % kStages2], (g / kStages2) & 1);
                            tc_fence_after();
                            const uint64_t dv = sdesc(smem_u32(sv + (g % kStages2) * kTileBytes), 16384, 1024);
    #pragma unroll
                            for (int k = 0; k < 8; ++k)
                                mma_ts_2sm(tO, tP + k * 8, dv + (uint64_t)(k << 7), id_o, (j > 0 || k > 0) ? 1u : 0u);
                            mbar_wait(&bars.p_full_hi, g & 1);
                            tc_fence_after();
    #pragma unroll
                            for (int k = 8; k < 16; ++k) mma_ts_2sm(tO, tP + k * 8, dv + (uint64_t)(k << 7), id_o, 1u);
                            mma_commit_2sm(&bars.o_full, 0x3);
                            mma_commit_2sm(&bars.v_empty[g % kStages2], 0x3);
                            // after the pair's last PV (so its epilogue starts as early as possible):
                            // the next pair's first S, which runs under that epilogue
                            if (j == it.jmax) {
                                nidx = take_pair(bars, n + 1, true);
                                if (nidx < a.pairs) {
                                    nit = pair_item(a, nidx, 0);
                                    mbar_wait(&bars.s_free, g & 1);
                                    mbar_wait(&bars.q_full[(n + 1) & 1], ((n + 1) >> 1) & 1);
                                    mbar_wait(&bars.k_full[(g + 1) % kStages2], ((g + 1) / kStages2) & 1);
                                    tc_fence_after();
                                    issue_s(g + 1, (n + 1) & 1, nit.jmax == 0);
                                }
                            }
                        }
                        if (nidx >= a.pairs) break;
                        it = nit;
                    }
                }
            }
        } else if (warp == kWStore) {
            // ------------------------------------------------------------ O stores (both CTAs)
            // The softmax warps stage each pair's normalised O tile in the pair's Q buffer (its
            // last S is done once O is final) in the SWIZZLE_128B layout of the Q boxes; two bulk
            // tensor stores write it (rows >= L clipped), then the buffer is released for the
            // Q of pair n + 2.
            if (elect_one()) {
                for (int n = 0;; ++n) {
                    const int idx = take_pair(bars, n, true);
                    if (idx >= a.pairs) break;
                    const Item it = pair_item(a, idx, (int)rank);
                    const int qb = n & 1;
                    mbar_wait(&bars.o_staged[qb], (n >> 1) & 1);
                    if (a.out && it.real) {
                        uint8_t* src = sq + qb * kTileBytes;
                        tma_store_3d(&to, src, 0, it.tile * kTile, it.plane);
                        tma_store_3d(&to, src + 16384, 64, it.tile * kTile, it.plane);
                        bulk_commit_group();
                        bulk_wait_group_read0();
                    }
                    mbar_arrive(&bars.q_empty[qb]);
                }
                bulk_wait_group0();
            }
        }
        teardown();
    } else {
        reg_alloc<kRegSoftmax>();
        // ---------------------------------------------------------------- softmax
        // warpgroup q owns key columns [32q, 32q + 32) of each 128-key half of S: every thread
        // computes its row's low-half keys first, stores them as P and signals, then the high half
        const int q = warp >> 2;
        const int wi = warp & 3;
        const int m = wi * 32 + (tid & 31);  // row within the CTA's tile
        const uint32_t lane_off = (uint32_t)(wi * 32) << 16;
        const uint32_t sS = tS + lane_off + 32 * q;  // + 128 for the high half
        const uint32_t sP = tP + lane_off + 16 * q;  // + 64 for the high half
        const uint32_t sO = tO + lane_off + 32 * q;
        // the leader's s_free, p_full, p_full_hi (adjacent barriers: one base register)
        const uint32_t s_free_l = mapa(smem_u32(&bars.s_free), 0);
        static_assert(offsetof(Bars2, p_full) == offsetof(Bars2, s_free) + 8 &&
                          offsetof(Bars2, p_full_hi) == offsetof(Bars2, s_free) + 16,
                      "barrier layout");
        const uint32_t xch_a = smem_u32(xch);
        int n_x = 0;  // row exchanges so far (selects the xch buffer; identical across a row's quarters)
        int g = 0;    // 256-key tiles consumed so far
        int idx = take_pair(bars, 0, (tid & 31) == 0);
        for (int n = 0; idx < a.pairs; ++n) {
            Item it = pair_item(a, idx, (int)rank);
            const int qrow = it.tile * kTile + m;      // query position
            const bool store = it.real && qrow < a.L;  // rows >= L (TMA zero fill) are computed, never stored
            const int km0 = it.unit * a.nT2;
            float km_next = __ldg(a.kmax + km0);
            float m_ref = -INFINITY, l = 0.f, qn = 0.f;
            for (int j = 0; j <= it.jmax; ++j, ++g) {
                const float km_j = km_next;
                if (j < it.jmax) km_next = __ldg(a.kmax + km0 + j + 1);
                mbar_wait(&bars.s_full, g & 1);
                tc_fence_after();
                uint32_t r[2][32];
                tmem_ld32(sS, r[0]);
                tmem_ld32(sS + 128, r[1]);
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if ((tid & 31) == 0) mbar_arrive_cluster(s_free_l);  // S_g may be overwritten
                const int key0 = 2 * j * kTile + 32 * q;  // chunk c covers keys key0 + 128 c + [0, 32)
                if (key0 + 128 + 31 > qrow) {  // causal mask near the diagonal
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int x = 0; x < 32; ++x)
                            if (key0 + c * 128 + x > qrow) r[c][x] = __float_as_uint(-INFINITY);
                }
                // warp-uniform (the exchange below is a named barrier); the four warps sharing these
                // rows see the same rows, hence the same vote
                const bool skip = __all_sync(0xffffffffu, j > 0 && qn * km_j * a.c <= m_ref + kSkip);
                float corr = 1.f;
                bool warp_need = false;
                if (!skip) {
                    float hmv[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int x = 0; x < 32; x += 8)
#pragma unroll
                            for (int gg = 0; gg < 4; gg += 2) {
                                hmv[gg] = fmax3(hmv[gg], __uint_as_float(r[c][x + 2 * gg]),
                                                __uint_as_float(r[c][x + 2 * gg + 1]));
                                hmv[gg + 1] = fmax3(hmv[gg + 1], __uint_as_float(r[c][x + 2 * gg + 2]),
                                                    __uint_as_float(r[c][x + 2 * gg + 3]));
                            }
                    const float hm = fmax3(hmv[0], hmv[1], fmaxf(hmv[2], hmv[3]));
                    const uint32_t xs = xch_a + (n_x++ & 1) * 2048;
                    sts32(xs + 4 * (q * 128 + m), hm);
                    asm volatile("bar.sync %0, 128;" ::"r"(1 + wi) : "memory");  // the 4 warps sharing these rows
                    const float4 o4 = make_float4(lds32(xs + 4 * m), lds32(xs + 4 * (128 + m)),
                                                  lds32(xs + 4 * (256 + m)), lds32(xs + 4 * (384 + m)));
                    const float mx = fmax3(o4.x, o4.y, fmaxf(o4.z, o4.w));
                    const float mx2 = mx * a.c;
                    const bool need = mx2 > m_ref + kRescale2;
                    warp_need = __any_sync(0xffffffffu, need);
                    const float new_m = need ? mx2 : m_ref;
                    corr = need ? ex2(m_ref - new_m) : 1.f;
                    m_ref = new_m;
                    l *= corr;
                }
                const float2 c2 = make_float2(a.c, a.c), nm2 = make_float2(-m_ref, -m_ref);
                float2 rs2 = make_float2(0.f, 0.f);
                uint32_t pk[16];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
#pragma unroll
                    for (int x = 0; x < 16; ++x) {
                        const float2 arg = __ffma2_rn(
                            make_float2(__uint_as_float(r[c][2 * x]), __uint_as_float(r[c][2 * x + 1])), c2, nm2);
                        // 1 of 8 pairs as the FMA-pipe polynomial, the rest on MUFU (persistent kernel:
                        // -1.5 % P1 time, -1 % sustained step; all-MUFU was best for the one-pair-per-
                        // cluster kernel).  A masked key (-inf) comes out as 2^-125, not 0: < 1e-35 of
                        // any row sum.
                        const float2 p = (x & 7) == 0 ? ex2_poly2(arg) : make_float2(ex2(arg.x), ex2(arg.y));
                        rs2 = __fadd2_rn(rs2, p);
                        pk[x] = pack_bf16(p.x, p.y);
                    }
                    if (c == 0 && j > 0) {  // P region free and O stable once PV_{g-1} is done
                        mbar_wait(&bars.o_full, (g - 1) & 1);
                        tc_fence_after();
                        if (warp_need) {  // rescale this quarter of O (rare), before PV_g starts; 16
                                          // columns at a time (register peak)
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                uint32_t o[16];
                                tmem_ld16(sO + 16 * h, o);
                                tmem_ld_wait();
#pragma unroll
                                for (int x = 0; x < 16; ++x) o[x] = __float_as_uint(__uint_as_float(o[x]) * corr);
                                tmem_st16(sO + 16 * h, o);
                            }
                        }
                    }
                    tmem_st16(sP + 64 * c, pk);
                    tmem_st_wait();
                    tc_fence_before();
                    __syncwarp();
                    if ((tid & 31) == 0) mbar_arrive_cluster(s_free_l + 8 * (c + 1));  // p_full / p_full_hi
                }
                l += rs2.x + rs2.y;
                if (j == 0) {
                    // |q_row| for the logit bound of tiles >= 1, from this CTA's Q tile in shared
                    // memory (resident until this pair's O is stored from it): quarter q
                    // sums dims [32q, 32q + 32) (SWIZZLE_128B rows), the four partials combine in a
                    // fixed order.  Rows >= L are TMA zero fill.
                    const uint32_t qrow_a = smem_u32(sq + (n & 1) * kTileBytes) + (q >> 1) * 16384 + m * 128;
                    float ss = 0.f;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float4 w4 = lds128(qrow_a + ((((q & 1) * 4 + c) ^ (m & 7)) << 4));
                        const uint32_t wv[4] = {__float_as_uint(w4.x), __float_as_uint(w4.y), __float_as_uint(w4.z),
                                                __float_as_uint(w4.w)};
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            const float lo = __uint_as_float(wv[t] << 16), hi = __uint_as_float(wv[t] & 0xFFFF0000u);
                            ss = fmaf(lo, lo, fmaf(hi, hi, ss));
                        }
                    }
                    const uint32_t xs = xch_a + (n_x++ & 1) * 2048;
                    sts32(xs + 4 * (q * 128 + m), ss);
                    asm volatile("bar.sync %0, 128;" ::"r"(1 + wi) : "memory");  // the 4 warps sharing these rows
                    qn = sqrtf((lds32(xs + 4 * m) + lds32(xs + 4 * (128 + m))) +
                               (lds32(xs + 4 * (256 + m)) + lds32(xs + 4 * (384 + m)))) * 1.0001f;  // rounding margin
                }
            }
            // the next pair, before this pair's epilogue
            const int nidx = take_pair(bars, n + 1, (tid & 31) == 0);
            // epilogue: l = sum of the four quarters (fixed order), O / l -> bf16, LSE.  The next
            // pair's first S is computed meanwhile; its P (and so its first PV, which overwrites O)
            // waits for this warp's O read below.
            const uint32_t xs = xch_a + (n_x++ & 1) * 2048;
            sts32(xs + 4 * (q * 128 + m), l);
            asm volatile("bar.sync %0, 128;" ::"r"(1 + wi) : "memory");  // the 4 warps sharing these rows
            const float lt = ((lds32(xs + 4 * m) + lds32(xs + 4 * (128 + m))) + lds32(xs + 4 * (256 + m))) +
                             lds32(xs + 4 * (384 + m));
            mbar_wait(&bars.o_full, (g - 1) & 1);
            tc_fence_after();
            it = pair_item(a, idx, (int)rank);
            const size_t row = (size_t)it.plane * a.L + qrow;
            const float inv = 1.f / lt;
            if (a.out) {  // O / l -> bf16, staged in this pair's Q buffer for the store thread
                uint32_t o[32];
                tmem_ld32(sO, o);
                tmem_ld_wait();
                const uint32_t srow = smem_u32(sq + (n & 1) * kTileBytes) + (q >> 1) * 16384 + m * 128;
#pragma unroll
                for (int x = 0; x < 4; ++x)
                    sts128(srow + ((((q & 1) * 4 + x) ^ (m & 7)) << 4),
                           pack_bf16(__uint_as_float(o[8 * x + 0]) * inv, __uint_as_float(o[8 * x + 1]) * inv),
                           pack_bf16(__uint_as_float(o[8 * x + 2]) * inv, __uint_as_float(o[8 * x + 3]) * inv),
                           pack_bf16(__uint_as_float(o[8 * x + 4]) * inv, __uint_as_float(o[8 * x + 5]) * inv),
                           pack_bf16(__uint_as_float(o[8 * x + 6]) * inv, __uint_as_float(o[8 * x + 7]) * inv));
                fence_proxy_async();  // generic-proxy stores -> visible to the bulk store (async proxy)
            }
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(&bars.o_staged[n & 1]);
            tc_fence_before();
            if (q == 0 && store) {
                const float lse2 = m_ref + __log2f(lt);
                // P2 folds the row normalisation into its MMA: Q' = [q, x1, x2, x3, 0...] against
                // K' = [k, 1, ..., 1] gives q.k + x with x = -lse2 / c, so S' c = s c - lse2 exactly
                // to fp32 rounding (three bf16 terms carry x to ~1e-6 absolute)
                const float x = -lse2 / a.c;
                const __nv_bfloat16 x1 = __float2bfloat16_rn(x);
                const float r1 = x - __bfloat162float(x1);
                const __nv_bfloat16 x2 = __float2bfloat16_rn(r1);
                const __nv_bfloat16 x3 = __float2bfloat16_rn(r1 - __bfloat162float(x2));
                uint4* dq = reinterpret_cast<uint4*>(a.qx + ((size_t)it.plane * a.Lp + qrow) * 16);
                const __nv_bfloat162 p12 = __halves2bfloat162(x1, x2), p30 = __halves2bfloat162(x3, __float2bfloat16_rn(0.f));
                dq[0] = make_uint4(*reinterpret_cast<const uint32_t*>(&p12), *reinterpret_cast<const uint32_t*>(&p30), 0u, 0u);
                dq[1] = make_uint4(0u, 0u, 0u, 0u);
                if (a.lse_nat) a.lse_nat[row] = lse2 * kLn2;
            }
            idx = nidx;
        }
        teardown();
    }
}

// max ||k|| over each 256-key tile of each unit (fp32): the per-tile logit bound of fwd2
// (and zeroes fwd2's scheduler counters, one per head part: the launches are stream-ordered)
__global__ void __launch_bounds__(256) key_tile_norm_kernel(const __nv_bfloat16* __restrict__ k, int L, int nT2,
                                                           float* __restrict__ kmax, int* __restrict__ next) {
    __shared__ float sh[8];
    if (blockIdx.x == 0 && threadIdx.x < 4) next[threadIdx.x] = 0;
    const int t = blockIdx.x % nT2, u = blockIdx.x / nT2;
    // a half-warp per key row (16 lanes x 16 bytes = the 256-byte row: fully coalesced), each
    // warp 32 rows of the tile, 4 rows per lane in flight
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, half = lane >> 4, c = lane & 15;
    const uint4* base = reinterpret_cast<const uint4*>(k + (size_t)u * L * kD) + c;
    float mx = 0.f;
#pragma unroll
    for (int it = 0; it < 16; it += 4) {
        uint4 w[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const int key = t * 256 + warp * 32 + 2 * (it + x) + half;
            w[x] = key < L ? base[(size_t)key * (kD / 8)] : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const uint32_t wv[4] = {w[x].x, w[x].y, w[x].z, w[x].w};
            float ss = 0.f;
#pragma unroll
            for (int y = 0; y < 4; ++y) {
                const float lo = __uint_as_float(wv[y] << 16), hi = __uint_as_float(wv[y] & 0xFFFF0000u);
                ss = fmaf(lo, lo, fmaf(hi, hi, ss));
            }
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);  // within the half
            mx = fmaxf(mx, sqrtf(ss));
        }
    }
    mx = warp_max(mx);
    if (lane == 0) sh[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = sh[0];
        for (int i = 1; i < 8; ++i) m = fmaxf(m, sh[i]);
        kmax[blockIdx.x] = m * 1.0001f;
    }
}

}  // namespace

// per-key-tile norm bounds, then the scheduler's counter
static size_t kmax_bytes(int units, int L) { return (sizeof(float) * (size_t)units * ((L + 255) / 256) + 255) / 256 * 256; }
size_t fwd2_workspace(int units, int L) { return kmax_bytes(units, L) + 256; }

bool fwd2_tc_supported(int L) { return (L + 255) / 256 <= kMaxT2; }

cudaError_t launch_fwd2_tc(int L, int Hq, int Hkv, int G, int units, float c, void* out, void* qx,
                           float* lse_nat, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                           const CUtensorMap& to,
                           const void* k, float* kmax, cudaStream_t s, int h0, int Gs, int part) {
    cudaError_t e = smem_optin(reinterpret_cast<const void*>(fwd2_tc_kernel), (int)kSmem2);
    if (e != cudaSuccess) return e;
    Fwd2Args a;
    a.L = L;
    a.nT = (L + kTile - 1) / kTile;
    a.Lp = a.nT * kTile;
    a.Hq = Hq;
    a.Hkv = Hkv;
    a.G = G;
    a.h0 = h0;
    a.Gs = Gs > 0 ? Gs : G;
    if (h0 < 0 || a.h0 + a.Gs > G || part < 0 || part >= 4) return cudaErrorInvalidValue;
    a.units = units;
    a.c = c;
    a.out = static_cast<__nv_bfloat16*>(out);
    a.qx = static_cast<__nv_bfloat16*>(qx);
    a.lse_nat = lse_nat;
    a.nT2 = (L + 255) / 256;
    a.kmax = kmax;
    const long long pairs = (long long)units * ((a.Gs * a.nT + 1) / 2);
    if (pairs >= (1ll << 30)) return cudaErrorInvalidValue;
    a.pairs = (int)pairs;
    a.next = reinterpret_cast<int*>(reinterpret_cast<char*>(kmax) + kmax_bytes(units, L)) + part;
    const int slots = active_clusters(reinterpret_cast<const void*>(fwd2_tc_kernel), kT2, (int)kSmem2, 2);
    const int clusters = (int)(pairs < slots ? pairs : slots);
    if (part == 0)  // the key bounds once per problem; it also zeroes the scheduler counters of every part
        key_tile_norm_kernel<<<units * a.nT2, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(k), L, a.nT2, kmax, a.next);
    fwd2_tc_kernel<<<(unsigned)(2 * clusters), kT2, kSmem2, s>>>(tq, tk, tv, to, a);
    return cudaGetLastError();
}

}  // namespace ems
