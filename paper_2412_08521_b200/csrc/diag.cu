// diag.cu -- the per-head diagnostics of analyze_trace (proj/src/experiment.cpp:133-150),
// SURVEY.md 8f row f4:
//
//   sparsity   = sparsity_rate(combine_glo_loc(glo, loc), zeta)   analysis.cpp:71-91,
//                                                                  scoring.cpp:105-124
//   redundancy = redundancy_rate_direct(k_raw, v_raw, tau)         analysis.cpp:93-118
//
// Sparsity (one 1024-thread CTA per unit): fp64 alignment sums and combined scores, each
// divided by the total once (the reference adds sorted[i] / total); the crossing value
// v = the largest score whose upper mass reaches zeta is found by a bitwise search over
// the fp64 bit patterns (63 passes of fixed-order block sums, deterministic), then the
// reference's sequential walk runs over the ties at v: needed = #(> v) + the first m with
// mass(> v) + m * v >= zeta.
//
// Redundancy: R[t][j] = clamp(cos(k_t, k_j)) * clamp(cos(v_t, v_j)) over j < t, token t
// counts when max_j R >= tau (t >= 1).  bf16 / head_dim 128 runs on the tensor cores (the
// similarity GEMMs of the merge step, causally tiled: one CTA per (unit, 128-row tile),
// column tiles 0..t streamed through a 2-stage TMA ring, K and V products in a
// double-buffered TMEM pair, masked max epilogue, integer counts); other shapes take a
// warp-per-token SIMT kernel.  Zero-norm tokens have similarity 0 (cos_or_zero,
// analysis.cpp:16-24) through a zero inverse norm.
#include <math.h>

#include "score_tc.cuh"
#include "tmap.h"

namespace ems {

namespace {

using namespace tc;
using namespace sc;

constexpr int kSpT = 1024;

__device__ double sp_sum(double v, double* sh) {  // fixed-order block sum
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double t = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    return warp_sum(t);
}

__device__ int sp_isum(int v, int* sh) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    int t = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    return t;
}

__global__ void __launch_bounds__(kSpT) sparsity_kernel(const float* __restrict__ glo,
                                                        const float* __restrict__ loc, int L,
                                                        double zeta, double* __restrict__ q_all,
                                                        double* __restrict__ rate, DevStatus* status,
                                                        int unit_base) {
    __shared__ double sh[32];
    __shared__ int shi[32];
    const int u = blockIdx.x, tid = threadIdx.x;
    const float* g = glo + (size_t)u * L;
    const float* lo = loc + (size_t)u * L;
    double* q = q_all + (size_t)u * L;
    // combine_glo_loc: align = sum(loc) / sum(glo) over all tokens, s = max(glo * align, loc)
    double sg = 0.0, sl = 0.0;
    for (int i = tid; i < L; i += kSpT) sg += (double)g[i], sl += (double)lo[i];
    sg = sp_sum(sg, sh);
    sl = sp_sum(sl, sh);
    if (!(sg > 0.0)) {  // DegenerateInputError (scoring.cpp:115-117)
        if (tid == 0) record_status(status, EMS_DEGENERATE_INPUT, unit_base + u), rate[u] = NAN;
        return;
    }
    const double align = sl / sg;
    double tot = 0.0;
    for (int i = tid; i < L; i += kSpT) {
        const double a = (double)g[i] * align, b = (double)lo[i];
        const double s = a > b ? a : b;
        q[i] = s;
        tot += s;
    }
    tot = sp_sum(tot, sh);
    if (!(tot > 0.0)) {  // "score has no mass" (analysis.cpp:77-79)
        if (tid == 0) record_status(status, EMS_DEGENERATE_INPUT, unit_base + u), rate[u] = NAN;
        return;
    }
    for (int i = tid; i < L; i += kSpT) q[i] = q[i] / tot;  // the per-element quotients the walk adds
    // bitwise search: v = max{key : mass(q >= key) >= zeta}; scores are >= 0, so the fp64
    // bit patterns order like the values and bit 63 is clear
    unsigned long long pre = 0ull;
    for (int bit = 62; bit >= 0; --bit) {
        const unsigned long long t = pre | (1ull << bit);
        double m = 0.0;
        for (int i = tid; i < L; i += kSpT) {
            const double x = q[i];
            if ((unsigned long long)__double_as_longlong(x) >= t) m += x;
        }
        m = sp_sum(m, sh);
        if (m >= zeta) pre = t;
    }
    double mg = 0.0;
    int cg = 0, ce = 0;
    for (int i = tid; i < L; i += kSpT) {
        const double x = q[i];
        const unsigned long long k = (unsigned long long)__double_as_longlong(x);
        if (k > pre) mg += x, ++cg;
        else if (k == pre) ++ce;
    }
    mg = sp_sum(mg, sh);
    cg = sp_isum(cg, shi);
    ce = sp_isum(ce, shi);
    if (tid == 0) {
        const double v = __longlong_as_double((long long)pre);
        long long needed = L;
        if (pre != 0ull) {
            double cum = mg;
            needed = min((long long)L, (long long)cg + ce + 1);  // rounding: the next token crosses
            for (int m = 1; m <= ce; ++m) {
                cum += v;
                if (cum >= zeta) {
                    needed = (long long)cg + m;
                    break;
                }
            }
        }
        rate[u] = 1.0 - (double)needed / (double)L;
    }
}

// Inverse norms of every token row of K and V (0 for zero rows), padded to 128 rows.
template <typename T>
__global__ void __launch_bounds__(256) inv_norm_kernel(const T* __restrict__ k, const T* __restrict__ v, int L,
                                                       int Lpad, int d, float* __restrict__ inv) {
    const int u = blockIdx.y;
    const int t = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (t >= Lpad) return;
    float sk = 0.f, sv = 0.f;
    if (t < L) {
        for (int x = lane; x < d; x += 32) {
            const float a = ld(k + ((size_t)u * L + t) * d + x), b = ld(v + ((size_t)u * L + t) * d + x);
            sk = fmaf(a, a, sk), sv = fmaf(b, b, sv);
        }
    }
    sk = warp_sum(sk), sv = warp_sum(sv);
    if (lane == 0) {
        inv[(size_t)u * 2 * Lpad + t] = sk > 0.f ? 1.f / sqrtf(sk) : 0.f;
        inv[(size_t)u * 2 * Lpad + Lpad + t] = sv > 0.f ? 1.f / sqrtf(sv) : 0.f;
    }
}

// SIMT: one warp per token t, lanes over d, all j < t.
template <typename T>
__global__ void __launch_bounds__(256) redundancy_simt_kernel(const T* __restrict__ k, const T* __restrict__ v,
                                                              int L, int Lpad, int d, const float* __restrict__ inv,
                                                              double tau, int* __restrict__ count) {
    const int u = blockIdx.y;
    const int t = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (t < 1 || t >= L) return;
    const float* ik = inv + (size_t)u * 2 * Lpad;
    const float* iv = ik + Lpad;
    const T* kb = k + (size_t)u * L * d;
    const T* vb = v + (size_t)u * L * d;
    float kt[4], vt[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int x = lane + 32 * e;
        kt[e] = x < d ? ld(kb + (size_t)t * d + x) : 0.f;
        vt[e] = x < d ? ld(vb + (size_t)t * d + x) : 0.f;
    }
    const float ikt = ik[t], ivt = iv[t];
    float best = -INFINITY;
    for (int j = 0; j < t; ++j) {
        float dk = 0.f, dv = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int x = lane + 32 * e;
            if (x < d) {
                dk = fmaf(kt[e], ld(kb + (size_t)j * d + x), dk);
                dv = fmaf(vt[e], ld(vb + (size_t)j * d + x), dv);
            }
        }
        dk = warp_sum(dk), dv = warp_sum(dv);
        const float ck = fminf(1.f, fmaxf(-1.f, dk * ikt * ik[j]));
        const float cv = fminf(1.f, fmaxf(-1.f, dv * ivt * iv[j]));
        best = fmaxf(best, ck * cv);
    }
    if (lane == 0 && (double)best >= tau) atomicAdd(count + u, 1);
}

// Tensor cores: one CTA per (unit, 128-token row tile), heaviest tiles first.
constexpr int kStages = 2;
static_assert(kStages == 2, "stage s of tile c is TMEM buffer c & 1 (the producer waits on d_empty[s])");
constexpr int kThreads = 384;  // w0 TMA, w1 MMA, w4-7 epilogue A, w8-11 epilogue B
constexpr size_t kSmem = 1024 + 2 * kTileBytes + kStages * (2 * kTileBytes + 1024) + 2 * 128 * 4;

struct RBars {
    uint64_t t_full;
    uint64_t c_full[kStages], c_empty[kStages];
    uint64_t d_full[2], d_empty[2];
    uint32_t tmem_base;
};

__global__ void __launch_bounds__(kThreads, 1)
    redundancy_tc_kernel(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv, int L,
                         int Lpad, const float* __restrict__ inv, double tau, int* __restrict__ count) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* skt = sm;
    uint8_t* svt = skt + kTileBytes;
    uint8_t* sring = svt + kTileBytes;  // stages x (K_c, V_c, inv_k[128], inv_v[128])
    float* sbest = reinterpret_cast<float*>(sring + kStages * (2 * kTileBytes + 1024));
    __shared__ RBars bars;

    const int tid = threadIdx.x, warp = tid >> 5;
    const int u = blockIdx.y;
    const int n_rt = Lpad / 128;
    const int rt = n_rt - 1 - (int)blockIdx.x;  // heaviest (most column tiles) first
    const int t0 = rt * 128;
    const int n_ct = rt + 1;
    const float* invu = inv + (size_t)u * 2 * Lpad;

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
            tma_load_3d(skt, &tk, &bars.t_full, 0, t0, u);
            tma_load_3d(skt + 16384, &tk, &bars.t_full, 64, t0, u);
            tma_load_3d(svt, &tv, &bars.t_full, 0, t0, u);
            tma_load_3d(svt + 16384, &tv, &bars.t_full, 64, t0, u);
            for (int c = 0; c < n_ct; ++c) {
                const int s = c % kStages;
                if (c >= kStages) {
                    mbar_wait(&bars.c_empty[s], ((c / kStages) - 1) & 1);
                    // the epilogue of tile c - 2 still reads this stage's column norms
                    mbar_wait(&bars.d_empty[s], ((c >> 1) - 1) & 1);
                }
                uint8_t* st = sring + s * (2 * kTileBytes + 1024);
                mbar_expect_tx(&bars.c_full[s], 2 * kTileBytes + 1024);
                tma_load_3d(st, &tk, &bars.c_full[s], 0, c * 128, u);
                tma_load_3d(st + 16384, &tk, &bars.c_full[s], 64, c * 128, u);
                tma_load_3d(st + kTileBytes, &tv, &bars.c_full[s], 0, c * 128, u);
                tma_load_3d(st + kTileBytes + 16384, &tv, &bars.c_full[s], 64, c * 128, u);
                bulk_load(st + 2 * kTileBytes, invu + c * 128, 512, &bars.c_full[s]);
                bulk_load(st + 2 * kTileBytes + 512, invu + Lpad + c * 128, 512, &bars.c_full[s]);
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
                    mma_ss(tmem + 256 * b, sdesc(kmajor_addr(ka, k), 16, 1024), sdesc(kmajor_addr(kc, k), 16, 1024),
                           id, k > 0);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    mma_ss(tmem + 256 * b + 128, sdesc(kmajor_addr(va, k), 16, 1024),
                           sdesc(kmajor_addr(vc, k), 16, 1024), id, k > 0);
                mma_commit(&bars.d_full[b]);
                mma_commit(&bars.c_empty[s]);
            }
        }
    } else if (warp >= 4) {
        const int g = (warp - 4) >> 2;  // epilogue warpgroup: column tiles c = g, g + 2, ...
        const int wi = warp & 3;
        const int row = wi * 32 + (tid & 31);
        const int t = t0 + row;
        const float ikt = invu[t], ivt = invu[Lpad + t];
        float best = -INFINITY;
        for (int c = g; c < n_ct; c += 2) {
            const int s = c % kStages, b = c & 1;
            mbar_wait(&bars.d_full[b], (c >> 1) & 1);
            tc_fence_after();
            const uint32_t ls = smem_u32(sring + s * (2 * kTileBytes + 1024) + 2 * kTileBytes);
            const uint32_t dk = tmem + 256 * b + ((uint32_t)(wi * 32) << 16);
            const int lim = c < rt ? 128 : row;  // causal: columns j < t only
#pragma unroll 1
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t rk[32], rv[32];
                tmem_ld32(dk + ch * 32, rk);
                tmem_ld32(dk + 128 + ch * 32, rv);
                tmem_ld_wait();
#pragma unroll
                for (int x = 0; x < 32; ++x) {
                    const float ck = fminf(1.f, fmaxf(-1.f, __uint_as_float(rk[x]) * ikt * lds32(ls + 4 * (ch * 32 + x))));
                    const float cv =
                        fminf(1.f, fmaxf(-1.f, __uint_as_float(rv[x]) * ivt * lds32(ls + 512 + 4 * (ch * 32 + x))));
                    if (ch * 32 + x < lim) best = fmaxf(best, ck * cv);
                }
            }
            tc_fence_before();
            mbar_arrive(&bars.d_empty[b]);
        }
        if (g == 1) sbest[row] = best;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (g == 0) {
            best = fmaxf(best, sbest[row]);
            const bool red = t >= 1 && t < L && (double)best >= tau;
            const unsigned m = __ballot_sync(0xffffffffu, red);
            if ((tid & 31) == 0 && m) atomicAdd(count + u, __popc(m));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

__global__ void rate_kernel(const int* __restrict__ count, int units, int L, double* __restrict__ rate) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < units) rate[u] = (double)count[u] / (double)L;
}

}  // namespace

// workspace: [status 256 B][sparsity quotients U*L f64][inverse norms U*2*Lpad f32][counts U i32]
struct DiagLayout {
    size_t q, inv, count, total;
    DiagLayout(int units, int L) {
        const size_t Lpad = (size_t)(L + 127) / 128 * 128;
        auto up = [](size_t x) { return (x + 255) / 256 * 256; };
        q = 256;
        inv = q + up((size_t)units * L * 8);
        count = inv + up((size_t)units * 2 * Lpad * 4);
        total = count + up((size_t)units * 4);
    }
};

size_t diag_workspace_bytes(int units, int L) { return DiagLayout(units, L).total; }

cudaError_t launch_sparsity(int units, int L, const float* glo, const float* loc, double zeta, double* rate,
                            void* ws, int unit_base, cudaStream_t s) {
    uint8_t* p = static_cast<uint8_t*>(ws);
    DevStatus* status = reinterpret_cast<DevStatus*>(p);
    double* q = reinterpret_cast<double*>(p + DiagLayout(units, L).q);
    cudaError_t e = cudaMemsetAsync(status, 0, sizeof(DevStatus), s);
    if (e != cudaSuccess) return e;
    sparsity_kernel<<<units, kSpT, 0, s>>>(glo, loc, L, zeta, q, rate, status, unit_base);
    return cudaGetLastError();
}

cudaError_t launch_redundancy(int units, int L, int d, int dtype, const void* k, const void* v, double tau,
                              double* rate, void* ws, cudaStream_t s) {
    const int Lpad = (L + 127) / 128 * 128;
    uint8_t* p = static_cast<uint8_t*>(ws);
    cudaError_t e = cudaMemsetAsync(p, 0, sizeof(DevStatus), s);
    if (e != cudaSuccess) return e;
    const DiagLayout lay(units, L);
    float* inv = reinterpret_cast<float*>(p + lay.inv);
    int* count = reinterpret_cast<int*>(p + lay.count);
    if ((e = cudaMemsetAsync(count, 0, (size_t)units * 4, s)) != cudaSuccess) return e;
    dim3 gn(Lpad / 8, units);
    if (dtype == EMS_F32)
        inv_norm_kernel<float><<<gn, 256, 0, s>>>((const float*)k, (const float*)v, L, Lpad, d, inv);
    else
        inv_norm_kernel<__nv_bfloat16><<<gn, 256, 0, s>>>((const __nv_bfloat16*)k, (const __nv_bfloat16*)v, L,
                                                          Lpad, d, inv);
    CUtensorMap tk, tv;
    const bool tc = dtype == EMS_BF16 && d == kD && L >= 128 && encode_fn() != nullptr && getenv("EMS_DIAG_SIMT") == nullptr &&
                    make_tmap_bf16_3d(&tk, k, kD, L, units, 128) && make_tmap_bf16_3d(&tv, v, kD, L, units, 128);
    if (tc) {
        const cudaError_t e = smem_optin(reinterpret_cast<const void*>(redundancy_tc_kernel), (int)kSmem);
        if (e != cudaSuccess) return e;
        redundancy_tc_kernel<<<dim3(Lpad / 128, units), kThreads, kSmem, s>>>(tk, tv, L, Lpad, inv, tau, count);
    } else {
        dim3 g((L + 7) / 8, units);
        if (dtype == EMS_F32)
            redundancy_simt_kernel<float><<<g, 256, 0, s>>>((const float*)k, (const float*)v, L, Lpad, d, inv, tau,
                                                            count);
        else
            redundancy_simt_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(
                (const __nv_bfloat16*)k, (const __nv_bfloat16*)v, L, Lpad, d, inv, tau, count);
    }
    rate_kernel<<<(units + 127) / 128, 128, 0, s>>>(count, units, L, rate);
    return cudaGetLastError();
}

}  // namespace ems
