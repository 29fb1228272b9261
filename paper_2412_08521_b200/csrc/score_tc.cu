// score_tc.cu -- host side of the tcgen05/TMEM/TMA score pass (bf16, head_dim 128, any L, any G).
//
// (P1) fwd2_tc.cu:   causal FlashAttention forward on CTA pairs (cta_group::2): O, row LSE.
// (P2) colsum_tc.cu: KV-stationary column sums (glo, loc) normalised with P1's LSE.
//
// Reference semantics: streaming_pass, proj/src/scoring.cpp:20-64 (prefill_attention /
// prefill_scores, scoring.cpp:86-103); GQA mean per contract D2.
#include <cuda.h>

#include "score_tc.cuh"
#include "tmap.h"

namespace ems {

using namespace sc;

bool score_tc_supported(const Dims& dm, int dtype) {
    if (dtype != EMS_BF16 || dm.d != kD || dm.L < 1 || !fwd2_tc_supported(dm.L)) return false;
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    return major == 10 && minor == 0 && encode_fn() != nullptr;
}

static int n_tiles(const Dims& dm) { return (dm.L + kTile - 1) / kTile; }

// workspace: qx [B*Hq][nT*128][16] bf16 (P1 -> P2: the row normalisation as extra K columns of
// Q, rows padded to whole tiles), then (head split only) fp64 partials [2][units][hsplit][L],
// then P1's per-key-tile norm bounds
static size_t qx_bytes(const Dims& dm) {
    return (32 * (size_t)dm.B * dm.Hq * n_tiles(dm) * kTile + 255) / 256 * 256;
}
static size_t part_bytes(const Dims& dm) {
    const int hs = colsum_hsplit(dm.G, n_tiles(dm), dm.units);
    return hs > 1 ? 2 * sizeof(double) * (size_t)dm.units * hs * dm.L : 0;
}
size_t score_tc_workspace(const Dims& dm) {
    return qx_bytes(dm) + part_bytes(dm) + (fwd2_workspace(dm.units, dm.L) + 255) / 256 * 256;
}

cudaError_t score_tc(const Dims& dm, const void* q, const void* k, const void* v, void* o,
                     float* lse, float* glo, float* loc, void* ws, cudaStream_t s, cudaEvent_t o_ready,
                     const ScoreParts* parts) {
    const int planes_q = dm.B * dm.Hq, planes_kv = dm.B * dm.Hkv;
    CUtensorMap tq, tk, tv;
    if (!make_tmap_bf16_3d(&tq, q, kD, dm.L, planes_q, kTile) ||
        !make_tmap_bf16_3d(&tk, k, kD, dm.L, planes_kv, kTile) ||
        !make_tmap_bf16_3d(&tv, v ? v : k, kD, dm.L, planes_kv, kTile))
        return cudaErrorInvalidValue;
    void* qx = ws;
    const float c = kLog2e / sqrtf((float)kD);
    float* kmax = reinterpret_cast<float*>(static_cast<char*>(ws) + qx_bytes(dm) + part_bytes(dm));
    CUtensorMap to = tq;  // O: the Q layout (only read when O is wanted)
    if (o && !make_tmap_bf16_3d(&to, o, kD, dm.L, planes_q, kTile)) return cudaErrorInvalidValue;
    cudaError_t e = cudaSuccess;
    const int np = parts && parts->n > 1 && dm.G % parts->n == 0 ? parts->n : 1;
    if (parts && np == 1)
        for (int p = 0; p < parts->n && e == cudaSuccess; ++p) e = parts->before(p, s);
    for (int p = 0; p < np && e == cudaSuccess; ++p) {
        if (np > 1) e = parts->before(p, s);
        if (e == cudaSuccess)
            e = launch_fwd2_tc(dm.L, dm.Hq, dm.Hkv, dm.G, dm.units, c, o, qx, lse, tq, tk, tv, to, k, kmax, s,
                               p * (dm.G / np), dm.G / np, p);
    }
    if (e != cudaSuccess) return e;
    if (o_ready && (e = cudaEventRecord(o_ready, s)) != cudaSuccess) return e;  // O and the LSE are final
    ColArgs ca;
    ca.L = dm.L;
    ca.Hq = dm.Hq;
    ca.Hkv = dm.Hkv;
    ca.G = dm.G;
    ca.nT = n_tiles(dm);
    ca.units = dm.units;
    ca.lwin = dm.lwin_scores;
    ca.c = c;
    ca.glo = glo;
    ca.loc = loc;
    ca.hsplit = colsum_hsplit(dm.G, ca.nT, dm.units);
    if (ca.hsplit > 1) {
        ca.part_g = reinterpret_cast<double*>(static_cast<char*>(ws) + qx_bytes(dm));
        ca.part_l = ca.part_g + (size_t)dm.units * ca.hsplit * dm.L;
    }
    CUtensorMap tq2, tqx;  // P2 streams pairs of query tiles (256-row boxes) and their qx rows
    if (!make_tmap_bf16_3d(&tq2, q, kD, dm.L, planes_q, 2 * kTile) ||
        !make_tmap_bf16_3d_k16(&tqx, qx, (uint64_t)ca.nT * kTile, planes_q, 2 * kTile))
        return cudaErrorInvalidValue;
    return launch_colsum_tc(ca, tk, tq2, tqx, s);
}

}  // namespace ems
