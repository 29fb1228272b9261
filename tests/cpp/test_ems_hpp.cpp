// test_ems_hpp.cpp -- TEST ONLY: the reference-shaped C++ API (include/ems_b200/ems.hpp)
// against the C restatement of the reference (oracle/ems_oracle.h) on seeded inputs.
// Exit code = number of failed checks.  Run by tests/test_gpu_cpp_api.py.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>

#include "ems_b200/ems.hpp"
#include "ems_oracle.h"

using namespace ems_b200;

static int g_fail = 0;
#define CHECK(cond, ...)                                          \
    do {                                                          \
        if (!(cond)) {                                            \
            ++g_fail;                                             \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__);      \
            std::printf(__VA_ARGS__);                             \
            std::printf("\n");                                    \
        }                                                         \
    } while (0)

static Matrix random_matrix(std::mt19937_64& gen, std::size_t r, std::size_t c) {
    std::normal_distribution<double> nd(0.0, 1.0);
    Matrix m(r, c);
    for (double& x : m.data) x = static_cast<double>(static_cast<float>(nd(gen)));  // fp32-exact
    return m;
}

static double max_rel(const Vector& a, const Vector& b, double floor = 1e-12) {
    double e = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i)
        e = std::max(e, std::abs(a[i] - b[i]) / std::max(std::abs(b[i]), floor));
    return e;
}

int main() {
    std::mt19937_64 gen(2024);
    const std::size_t n = 300, d = 64;
    const Matrix q = random_matrix(gen, n, d), k = random_matrix(gen, n, d), v = random_matrix(gen, n, d);

    // --- prefill_attention vs oracle (scoring.cpp:93-103)
    const PrefillAttention pa = prefill_attention(q, k, v, 32);
    Vector og(n), ol(n), oo(n * d), lse(n);
    ems_oracle_prefill_attention(q.data.data(), k.data.data(), v.data.data(), n, d, 32, oo.data(),
                                 og.data(), ol.data(), lse.data());
    CHECK(max_rel(pa.glo, og) < 2e-5, "glo rel err %g", max_rel(pa.glo, og));
    CHECK(max_rel(pa.loc, ol, 1e-6) < 2e-4, "loc rel err %g", max_rel(pa.loc, ol, 1e-6));
    CHECK(max_rel(pa.outputs.data, oo, 1e-3) < 1e-3, "O rel err %g", max_rel(pa.outputs.data, oo, 1e-3));

    // --- error behaviour mirrors the reference
    bool threw = false;
    try {
        local_score_prefill(q, k, n + 1);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw, "local_score_prefill(l_win > N) must throw invalid_argument");
    threw = false;
    try {
        combine_glo_loc(Vector{0.0, 0.0}, Vector{1.0, 1.0});
    } catch (const DegenerateInputError&) {
        threw = true;
    }
    CHECK(threw, "combine_glo_loc(zero mass) must throw DegenerateInputError");
    threw = false;
    try {
        compress_prefill(k, v, init_score_state(Vector(n - 1, 1.0), Vector(n - 1, 1.0), 8), {});
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw, "compress_prefill(inconsistent counts) must throw invalid_argument");

    // --- compress_prefill vs oracle on the oracle's own scores (compressor.cpp:163-242)
    CompressionConfig cfg;
    cfg.n_budget = 48;
    cfg.l_win = 8;
    cfg.gamma = 3.0;
    cfg.tau = 0.0;  // merges happen (every best R >= 0 merges)
    cfg.kernel_size = 5;
    const HeadCacheState hc = compress_prefill(k, v, init_score_state(og, ol, cfg.l_win), cfg);
    ems_oracle_config oc{48, 8, 0.0, 3.0, 0.95, 5, 1, 0};
    std::vector<double> uk(40 * d), kn(40), val(40 * d), sc(40 * 3), lk(48 * d), lv(48 * d), ls(48 * 3);
    std::vector<int64_t> pos(40), lpos(48), lutp(200);
    std::vector<int32_t> luts(200);
    ems_oracle_cache ref{(int64_t)d, 0, 0, uk.data(), kn.data(), val.data(), pos.data(), sc.data(), 0,
                         lk.data(), lv.data(), lpos.data(), ls.data(), 0, lutp.data(), luts.data()};
    Vector zeros(n, 0.0);
    ems_oracle_compress_prefill(k.data.data(), v.data.data(), og.data(), ol.data(), zeros.data(), n, d,
                                &oc, 0, &ref, nullptr, nullptr, nullptr);
    CHECK(hc.compressed && ref.compressed, "compressed flag");
    CHECK(hc.slots.size() == (std::size_t)ref.n_centers, "centers %zu vs %lld", hc.slots.size(),
          (long long)ref.n_centers);
    CHECK(hc.lut.size() == (std::size_t)ref.n_lut, "lut %zu vs %lld", hc.lut.size(), (long long)ref.n_lut);
    int lut_mismatch = 0;
    for (std::size_t i = 0; i < std::min(hc.lut.size(), (std::size_t)ref.n_lut); ++i)
        lut_mismatch += hc.lut[i].position != lutp[i] || hc.lut[i].slot != luts[i];
    CHECK(lut_mismatch == 0, "%d LUT entries differ", lut_mismatch);
    double vmax = 0.0;
    for (std::size_t s = 0; s < std::min(hc.slots.size(), (std::size_t)ref.n_centers); ++s) {
        CHECK(hc.slots[s]->position == pos[s], "slot %zu position", s);
        double num = 0.0, den = 0.0;
        for (std::size_t x = 0; x < d; ++x) {
            num += std::pow(hc.slots[s]->value[x] - val[s * d + x], 2);
            den += val[s * d + x] * val[s * d + x];
        }
        vmax = std::max(vmax, std::sqrt(num / den));
    }
    CHECK(vmax < 1e-4, "merged value rel err %g", vmax);

    // --- redundancy_cross (analysis.cpp:51-69)
    const Matrix kr = random_matrix(gen, 17, d), vr = random_matrix(gen, 17, d);
    const Matrix r = redundancy_cross(kr, vr, k, v);
    std::vector<double> rr(17 * n);
    ems_oracle_redundancy_cross(kr.data.data(), vr.data.data(), 17, k.data.data(), v.data.data(), n, d, 0,
                                rr.data());
    double re = 0.0;
    for (std::size_t i = 0; i < rr.size(); ++i) re = std::max(re, std::abs(r.data[i] - rr[i]));
    CHECK(re < 1e-5, "redundancy abs err %g", re);

    // --- diagnostics (analysis.cpp:71-118) vs the oracle restatement
    {
        Vector sc(300);
        for (std::size_t i = 0; i < sc.size(); ++i) sc[i] = (double)(float)(0.001 + (double)((i * 7919) % 997) / 997.0);
        for (double zeta : {0.1, 0.5, 0.95}) {
            double want = 0.0;
            ems_oracle_sparsity_rate(sc.data(), (int64_t)sc.size(), zeta, &want);
            CHECK(sparsity_rate(sc, zeta) == want, "sparsity_rate zeta %g", zeta);
        }
        bool threw = false;
        try {
            sparsity_rate(Vector(8, 0.0), 0.5);
        } catch (const DegenerateInputError&) {
            threw = true;
        }
        CHECK(threw, "sparsity_rate of a zero score must throw DegenerateInputError");
        double want_r = 0.0;
        const double got_r = redundancy_rate_direct(k, v, 0.2);
        ems_oracle_redundancy_rate_direct(k.data.data(), v.data.data(), (int64_t)n, (int64_t)d, 0.2, &want_r);
        CHECK(std::abs(got_r - want_r) * n <= 1.0, "redundancy_rate_direct %g vs %g", got_r, want_r);
    }

    // --- baseline policies (policies.cpp:131-180) vs the oracle restatement
    {
        const PolicyKind kinds[] = {PolicyKind::full, PolicyKind::streaming_llm, PolicyKind::h2o,
                                    PolicyKind::snapkv};
        const int codes[] = {EMS_ORACLE_POLICY_FULL, EMS_ORACLE_POLICY_STREAMING, EMS_ORACLE_POLICY_H2O,
                             EMS_ORACLE_POLICY_SNAPKV};
        std::vector<double> lk2(n * d), lv2(n * d), ls2(n * 3);
        std::vector<int64_t> lpos2(n);
        for (int pi = 0; pi < 4; ++pi) {
            PolicyHandle ph{kinds[pi], 4};
            const HeadCacheState got = policy_prefill_compress(ph, k, v, init_score_state(og, ol, cfg.l_win), cfg);
            ems_oracle_cache want{(int64_t)d, 0, 0, uk.data(), kn.data(), val.data(), pos.data(), sc.data(), 0,
                                  lk2.data(), lv2.data(), lpos2.data(), ls2.data(), 0, lutp.data(), luts.data()};
            ems_oracle_policy_prefill(codes[pi], 4, k.data.data(), v.data.data(), og.data(), ol.data(),
                                      zeros.data(), n, d, &oc, &want, nullptr);
            CHECK(got.slots.size() == (std::size_t)want.n_centers && got.locals.size() == (std::size_t)want.n_locals &&
                      got.lut.size() == (std::size_t)want.n_lut,
                  "policy %d sizes", pi);
            int mism = 0;
            for (std::size_t s = 0; s < std::min(got.slots.size(), (std::size_t)want.n_centers); ++s)
                mism += got.slots[s]->position != pos[s];
            for (std::size_t e = 0; e < std::min(got.lut.size(), (std::size_t)want.n_lut); ++e)
                mism += got.lut[e].position != lutp[e] || got.lut[e].slot != luts[e];
            CHECK(mism == 0, "policy %d: %d kept/LUT entries differ", pi, mism);
        }
        bool threw_p = false;
        try {
            CompressionConfig tight = cfg;
            tight.n_budget = 10;
            policy_prefill_compress(PolicyHandle{PolicyKind::streaming_llm, 4}, k, v,
                                    init_score_state(og, ol, tight.l_win), tight);
        } catch (const std::invalid_argument&) {
            threw_p = true;
        }
        CHECK(threw_p, "streaming_llm with n_budget < sinks + l_win must throw invalid_argument");
    }

    // --- engine-level prefill with GQA (G = 2), bf16 on device
    std::vector<Matrix> qs{q, random_matrix(gen, n, d)}, ks{k}, vs{v};
    const PrefillResult pr = prefill(qs, ks, ks, vs, cfg, EMS_BF16);
    CHECK(pr.outputs.size() == 2 && pr.heads.size() == 1 && pr.compression_applied, "prefill shapes");
    CHECK(pr.heads[0].slots.size() == cfg.center_capacity(), "prefill centers");

    std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "ok", g_fail);
    return g_fail;
}
