// score_tc.cuh -- constants and helpers shared by the tcgen05 score kernels.
#pragma once

#include <cuda.h>
#include <stdint.h>

#include "common.cuh"
#include "tc.cuh"

namespace ems {
namespace sc {

constexpr int kD = 128;                       // head_dim
constexpr int kTile = 128;                    // rows per Q / K / V tile
constexpr int kTileBytes = kTile * kD * 2;    // 32 KB = two 16 KB SWIZZLE_128B boxes
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// smem operand address of K-step k (16 elements) for a K-major 128x128 SW128 tile:
// elements [0,64) live in the first 16 KB box, [64,128) in the second.
__device__ __forceinline__ uint32_t kmajor_addr(uint32_t base, int k) {
    return base + (k >> 2) * 16384 + (k & 3) * 32;
}

// TMEM address of the warp's 32-lane subpartition (warp w % 4 owns lanes 32*(w%4)...).
__device__ __forceinline__ uint32_t tmem_lane_addr(uint32_t base, int warp_in_wg) {
    return base + ((uint32_t)(warp_in_wg * 32) << 16);
}

struct ColArgs {
    int L, Hq, Hkv, G, nT, units, lwin;
    float c;               // log2(e) / sqrt(d)
    float* glo;            // [units][L]
    float* loc;
    // Head split (load balance when few units): each CTA takes G / hsplit query heads of its
    // key-tile pair and writes fp64 partial sums part_{g,l}[unit][hsplit][L]; a reduce kernel
    // sums them in head-group order.  hsplit == 1 writes glo/loc directly.
    int hsplit = 1;
    double* part_g = nullptr;
    double* part_l = nullptr;
};

}  // namespace sc

cudaError_t launch_colsum_tc(const sc::ColArgs& a, const CUtensorMap& tk, const CUtensorMap& tq,
                             const CUtensorMap& tqx, cudaStream_t s);
int colsum_hsplit(int G, int nT, int units);
bool fwd2_tc_supported(int L);
size_t fwd2_workspace(int units, int L);
cudaError_t launch_fwd2_tc(int L, int Hq, int Hkv, int G, int units, float c, void* out, void* qx,
                           float* lse_nat, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                           const CUtensorMap& to,
                           const void* k, float* kmax, cudaStream_t s, int h0 = 0, int Gs = 0, int part = 0);

}  // namespace ems
