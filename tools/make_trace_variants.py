"""Build the instrumented variants the trace probes read (tools only, not the product):

    python tools/make_trace_variants.py      # -> _variants/p1trace.so, _variants/p2trace.so

p1trace: P1 records %globaltimer per pair (pair start, first S ready, last PV done, end) and the
SM id (tools/p1_trace_probe.py).  p2trace: P2 records per CTA start, first S, loop end, combine
done, exit (tools/p2_trace_probe.py).  The records go to a __device__ array read back through
an extra exported function; the kernels are otherwise the working tree's."""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2412_08521_b200", "csrc")


def sub(s, old, new):
    if old not in s:
        raise SystemExit(f"instrumentation anchor not found: {old[:60]!r}")
    return s.replace(old, new, 1)


TIMER = """__device__ __forceinline__ unsigned long long gtime_() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
"""


def p1():
    s = open(os.path.join(CSRC, "fwd2_tc.cu")).read()
    s = sub(s, "struct Fwd2Args {", "__device__ unsigned long long g_trace[1 << 17][6];\n" + TIMER + "struct Fwd2Args {")
    s = sub(s, """        for (int n = 0; idx < a.pairs; ++n) {
            Item it = pair_item(a, idx, (int)rank);""", """        for (int n = 0; idx < a.pairs; ++n) {
            if (tid == 0 && rank == 0) g_trace[idx][0] = gtime_();
            Item it = pair_item(a, idx, (int)rank);""")
    s = sub(s, """                mbar_wait(&bars.s_full, g & 1);
                tc_fence_after();""", """                mbar_wait(&bars.s_full, g & 1);
                if (j == 0 && tid == 0 && rank == 0) g_trace[idx][1] = gtime_();
                tc_fence_after();""")
    s = sub(s, """            mbar_wait(&bars.o_full, (g - 1) & 1);
            tc_fence_after();""", """            mbar_wait(&bars.o_full, (g - 1) & 1);
            if (tid == 0 && rank == 0) g_trace[idx][2] = gtime_();
            tc_fence_after();""")
    s = sub(s, """            idx = nidx;
        }
        teardown();""", """            if (tid == 0 && rank == 0) {
                unsigned smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                g_trace[idx][3] = g_trace[idx][4] = gtime_();
                g_trace[idx][5] = ((unsigned long long)smid << 32) | (unsigned)it.jmax;
            }
            idx = nidx;
        }
        teardown();""")
    s = sub(s, "bool fwd2_tc_supported(int L)", """extern "C" __attribute__((visibility("default"))) int ems_debug_fwd2_trace(void* host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, g_trace, bytes);
}

bool fwd2_tc_supported(int L)""")
    return "fwd2_tc.cu", s


def p2():
    s = open(os.path.join(CSRC, "colsum_tc.cu")).read()
    s = sub(s, "struct Bars {", "__device__ unsigned long long g_ctrace[1 << 16][5];\n" + TIMER + "struct Bars {")
    s = sub(s, """    const int tid = threadIdx.x, warp = tid >> 5;
    const int per_jp = a.units * a.hsplit;""", """    const unsigned long long t_start = gtime_();
    const int tid = threadIdx.x, warp = tid >> 5;
    const int per_jp = a.units * a.hsplit;""")
    s = sub(s, """                mbar_wait_u(s_full0 + 8 * w, p & 1);
                tc_fence_after();""", """                mbar_wait_u(s_full0 + 8 * w, p & 1);
                if (p == 0 && w == 0 && tid == 128) { g_ctrace[blockIdx.x][0] = t_start; g_ctrace[blockIdx.x][1] = gtime_(); }
                tc_fence_after();""")
    s = sub(s, "        // combine the four column quarters of each key tile in a fixed order",
            "        if (tid == 128) g_ctrace[blockIdx.x][2] = gtime_();\n"
            "        // combine the four column quarters of each key tile in a fixed order")
    s = sub(s, """    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}""", """    tc_fence_before();
    if (tid == 128) g_ctrace[blockIdx.x][3] = gtime_();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
    if (tid == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_ctrace[blockIdx.x][4] = ((unsigned long long)smid << 40) | (gtime_() & 0xFFFFFFFFFFull);
    }
}
}  // namespace
extern "C" __attribute__((visibility("default"))) int ems_debug_colsum_trace(void* host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, g_ctrace, bytes);
}
namespace {""")
    return "colsum_tc.cu", s


def main():
    for name, make in (("p1trace", p1), ("p2trace", p2)):
        fname, src = make()
        tmp = os.path.join(tempfile.mkdtemp(prefix=f"trace_{name}_"), fname)
        open(tmp, "w").write(src)
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "build_variant.py"), name, f"{fname}={tmp}"],
                       check=True)


if __name__ == "__main__":
    main()
