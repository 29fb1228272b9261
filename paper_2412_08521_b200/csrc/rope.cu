// rope.cu -- interleaved-pair rotary position embedding on the device.
//
// Restates detail::rotate (proj/src/rope.cpp:10-28) as engine::prefill applies it to every
// token of a prompt (rotate_block, proj/src/engine.cpp:14-22, 68-69): pair (2i, 2i+1) of the
// token at position p is rotated by  angle = p * base^(-2i/d)  with
//     y0 = x0*cos - x1*sin,   y1 = x0*sin + x1*cos
// evaluated in fp64 exactly as the reference does (separate products, no FMA contraction),
// then rounded once to the storage dtype (fp64 -> fp32 -> bf16, the same rounding the
// oracle's inputs use).  HBM-bound: one read and one write of the tensor; the fp64
// cos/sin of a (position, pair) are computed once and reused across all planes (heads).
#include "common.cuh"

namespace ems {

namespace {

template <typename T>
struct Pair;
template <>
struct Pair<float> {
    using V = float2;
    static __device__ __forceinline__ void get(V v, double& a, double& b) {
        a = v.x;
        b = v.y;
    }
    static __device__ __forceinline__ V make(double a, double b) {
        return make_float2((float)a, (float)b);
    }
};
template <>
struct Pair<__nv_bfloat16> {
    using V = __nv_bfloat162;
    static __device__ __forceinline__ void get(V v, double& a, double& b) {
        a = (double)__bfloat162float(v.x);
        b = (double)__bfloat162float(v.y);
    }
    static __device__ __forceinline__ V make(double a, double b) {
        // fp64 -> fp32 (RNE) -> bf16 (RNE): the oracle's round_to
        return __floats2bfloat162_rn((float)a, (float)b);
    }
};

constexpr int kThreads = 256;
constexpr int kUnroll = 4;  // planes in flight per thread

// x, y: [planes][L][d]; one thread = one (row, pair), looping over all planes.
template <typename T>
__global__ void __launch_bounds__(kThreads) rope_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                       int planes, int L, int d, double base,
                                                       long long first_pos) {
    using P = Pair<T>;
    using V = typename P::V;
    const int pairs = d / 2;
    const int rows_per_block = kThreads / pairs;
    const int j = threadIdx.x % pairs;
    const int l = blockIdx.x * rows_per_block + threadIdx.x / pairs;
    if (threadIdx.x >= rows_per_block * pairs || l >= L) return;
    const double freq = pow(base, -(double)(2 * j) / (double)d);
    const double angle = (double)(first_pos + l) * freq;
    double s, c;
    sincos(angle, &s, &c);
    const size_t plane_stride = (size_t)L * pairs;  // in pairs
    const V* xp = reinterpret_cast<const V*>(x) + (size_t)l * pairs + j;
    V* yp = reinterpret_cast<V*>(y) + (size_t)l * pairs + j;
    int p = 0;
    for (; p + kUnroll <= planes; p += kUnroll) {
        V v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) v[u] = xp[(size_t)(p + u) * plane_stride];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            double a, b;
            P::get(v[u], a, b);
            const double y0 = __dsub_rn(__dmul_rn(a, c), __dmul_rn(b, s));
            const double y1 = __dadd_rn(__dmul_rn(a, s), __dmul_rn(b, c));
            yp[(size_t)(p + u) * plane_stride] = P::make(y0, y1);
        }
    }
    for (; p < planes; ++p) {
        double a, b;
        P::get(xp[(size_t)p * plane_stride], a, b);
        const double y0 = __dsub_rn(__dmul_rn(a, c), __dmul_rn(b, s));
        const double y1 = __dadd_rn(__dmul_rn(a, s), __dmul_rn(b, c));
        yp[(size_t)p * plane_stride] = P::make(y0, y1);
    }
}

// The same rotation with (cos, sin) from a table computed once per problem (the fp64 pow and
// sincos dominate a launch over few planes: ~33 us of a 36 us one-plane launch at L = 32768).
template <typename T>
__global__ void __launch_bounds__(kThreads) rope_tab_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                           int planes, int L, int d,
                                                           const double2* __restrict__ tab) {
    using P = Pair<T>;
    using V = typename P::V;
    const int pairs = d / 2;
    const int rows_per_block = kThreads / pairs;
    const int j = threadIdx.x % pairs;
    const int l = blockIdx.x * rows_per_block + threadIdx.x / pairs;
    if (threadIdx.x >= rows_per_block * pairs || l >= L) return;
    const double2 cs = tab[(size_t)l * pairs + j];
    const double c = cs.x, s = cs.y;
    const size_t plane_stride = (size_t)L * pairs;  // in pairs
    const V* xp = reinterpret_cast<const V*>(x) + (size_t)l * pairs + j;
    V* yp = reinterpret_cast<V*>(y) + (size_t)l * pairs + j;
    int p = 0;
    for (; p + kUnroll <= planes; p += kUnroll) {
        V v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) v[u] = xp[(size_t)(p + u) * plane_stride];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            double a, b;
            P::get(v[u], a, b);
            const double y0 = __dsub_rn(__dmul_rn(a, c), __dmul_rn(b, s));
            const double y1 = __dadd_rn(__dmul_rn(a, s), __dmul_rn(b, c));
            yp[(size_t)(p + u) * plane_stride] = P::make(y0, y1);
        }
    }
    for (; p < planes; ++p) {
        double a, b;
        P::get(xp[(size_t)p * plane_stride], a, b);
        const double y0 = __dsub_rn(__dmul_rn(a, c), __dmul_rn(b, s));
        const double y1 = __dadd_rn(__dmul_rn(a, s), __dmul_rn(b, c));
        yp[(size_t)p * plane_stride] = P::make(y0, y1);
    }
}

// tab[l][j] = (cos, sin) of (first_pos + l) * base^(-2j/d), exactly as rope_kernel evaluates them
__global__ void rope_table64_kernel(double2* __restrict__ tab, int L, int d, double base, long long first_pos) {
    const int pairs = d / 2;
    const size_t n = (size_t)L * pairs;
    for (size_t x = blockIdx.x * (size_t)blockDim.x + threadIdx.x; x < n; x += (size_t)gridDim.x * blockDim.x) {
        const int j = (int)(x % pairs);
        const int l = (int)(x / pairs);
        const double freq = pow(base, -(double)(2 * j) / (double)d);
        const double angle = (double)(first_pos + l) * freq;
        double s, c;
        sincos(angle, &s, &c);
        tab[x] = make_double2(c, s);
    }
}

}  // namespace

size_t rope_table64_bytes(int L, int d) { return (size_t)L * (d / 2) * sizeof(double2); }

cudaError_t launch_rope_table64(void* tab, int L, int d, double base, long long first_pos, cudaStream_t s) {
    if (L <= 0) return cudaSuccess;
    rope_table64_kernel<<<8 * 148, 256, 0, s>>>(static_cast<double2*>(tab), L, d, base, first_pos);
    return cudaGetLastError();
}

cudaError_t launch_rope_tab(int dtype, int planes, int L, int d, const void* tab, const void* x, void* y,
                            cudaStream_t s) {
    if (planes <= 0 || L <= 0) return cudaSuccess;
    const int rows_per_block = kThreads / (d / 2);
    const dim3 grid((L + rows_per_block - 1) / rows_per_block);
    const double2* t = static_cast<const double2*>(tab);
    if (dtype == EMS_F32)
        rope_tab_kernel<float><<<grid, kThreads, 0, s>>>(static_cast<const float*>(x), static_cast<float*>(y), planes,
                                                         L, d, t);
    else
        rope_tab_kernel<__nv_bfloat16><<<grid, kThreads, 0, s>>>(static_cast<const __nv_bfloat16*>(x),
                                                                 static_cast<__nv_bfloat16*>(y), planes, L, d, t);
    return cudaGetLastError();
}

cudaError_t launch_rope(int dtype, int planes, int L, int d, double base, long long first_pos,
                        const void* x, void* y, cudaStream_t s) {
    if (planes <= 0 || L <= 0) return cudaSuccess;
    const int rows_per_block = kThreads / (d / 2);
    const dim3 grid((L + rows_per_block - 1) / rows_per_block);
    if (dtype == EMS_F32)
        rope_kernel<float><<<grid, kThreads, 0, s>>>(static_cast<const float*>(x), static_cast<float*>(y),
                                                     planes, L, d, base, first_pos);
    else
        rope_kernel<__nv_bfloat16><<<grid, kThreads, 0, s>>>(static_cast<const __nv_bfloat16*>(x),
                                                             static_cast<__nv_bfloat16*>(y), planes, L, d,
                                                             base, first_pos);
    return cudaGetLastError();
}

}  // namespace ems
