// The C++ adapter of INTEGRATION.md, compiled and run: a GpuStage owned next to the reference's
// StrategyContext replaces trace_frame's decision block (wavefront.cpp:363-425) with one
// nrrs_gpu_rrs_stage_host call per depth.  Built against the REFERENCE's own headers and
// rrs.cpp / networks.cpp / mlp.cpp / hashgrid.cpp (Eigen subset shim, oracle/eigen_shim) by
// tests/cpp/Makefile; the checks use the reference's own functions on the same inputs:
//   * NeuralRrs::load_checkpoint (networks.cpp:641-705) reads the snapshot this test was handed;
//   * predict_q per vertex (networks.cpp:266-281) vs the GPU's q_orig: within 1e-3 relative;
//   * normalize_factors (rrs.cpp:8-24) on the GPU's q_orig: the same float(F) and q_norm bit for bit;
//   * RateControl::gain (rrs.hpp:23-36) and realize_counts (rrs.cpp:35-45) on the GPU's u:
//     the same counts, total and queue offsets (plan_spawns' clip, wavefront.cpp:141-154).
// usage: gpu_stage_adapter <checkpoint> <variant 0|1> <n> -> exit 0 when every check holds
#include "nrrs/networks.hpp"
#include "nrrs/rng.hpp"
#include "nrrs/rrs.hpp"
#include "nrrs_gpu.h"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <vector>

struct GpuStage {  // owned next to the StrategyContext (wavefront.hpp:154-157)
    nrrs_gpu_ctx *ctx = nullptr;
    explicit GpuStage(int device) {
        if (nrrs_gpu_create(device, &ctx))
            throw std::runtime_error("nrrs_gpu_create failed");
    }
    ~GpuStage() { nrrs_gpu_destroy(ctx); }
    void check(int rc) {
        if (rc)
            throw std::runtime_error(nrrs_gpu_last_error(ctx));
    }
    void set_weights(const nrrs::NeuralRrs &nets) {  // the published snapshot (networks.cpp:199-204)
        const auto &cfg = nets.config();
        nrrs_net_weights w{};
        w.variant = cfg.variant == nrrs::RrsVariant::Aid ? NRRS_VARIANT_AID : NRRS_VARIANT_NRRS;
        w.grid = {cfg.grid.levels, cfg.grid.features, cfg.grid.base_resolution, cfg.grid.log2_table_size};
        w.stat_grid = nets.stat_grid().theta().data();
        w.stat_grid_len = (uint64_t)nets.stat_grid().theta().size();
        w.stat_mlp = nets.stat_mlp().theta().data();
        w.stat_mlp_len = (uint64_t)nets.stat_mlp().theta().size();
        w.rrs_grid = cfg.variant == nrrs::RrsVariant::Aid ? nets.rrs_grid().theta().data() : nullptr;
        w.rrs_grid_len = cfg.variant == nrrs::RrsVariant::Aid ? (uint64_t)nets.rrs_grid().theta().size() : 0;
        w.rrs_mlp = nets.rrs_mlp().theta().data();
        w.rrs_mlp_len = (uint64_t)nets.rrs_mlp().theta().size();
        check(nrrs_gpu_set_weights(ctx, &w));
    }
};

static int failures = 0;
#define EXPECT(c, ...)                                   \
    do {                                                 \
        if (!(c)) {                                      \
            std::fprintf(stderr, "FAIL: " __VA_ARGS__); \
            std::fprintf(stderr, "\n");                  \
            ++failures;                                  \
        }                                                \
    } while (0)

int main(int argc, char **argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: %s <checkpoint> <variant 0|1> <n>\n", argv[0]);
        return 2;
    }
    const int variant = std::atoi(argv[2]);
    const uint32_t n = (uint32_t)std::atoi(argv[3]);
    nrrs::NeuralRrsConfig cfg;
    cfg.variant = variant == 1 ? nrrs::RrsVariant::Aid : nrrs::RrsVariant::Nrrs;
    nrrs::NeuralRrs nets(cfg);
    nets.load_checkpoint(argv[1]);  // live == EMA == snapshot in the handed checkpoint

    // one depth's surface vertices, SURVEY.md 8d generator (RngStream(0xC0FFEE, i) per vertex)
    std::vector<float> p01(3 * n), wo01(2 * n), rough(n), weight(3 * n), ipix(3 * n);
    std::vector<uint64_t> keys(n);
    for (uint32_t i = 0; i < n; ++i) {
        nrrs::RngStream g(0xC0FFEE, i);
        for (int a = 0; a < 3; ++a) p01[3 * i + a] = g.next_float();
        for (int a = 0; a < 2; ++a) wo01[2 * i + a] = g.next_float();
        rough[i] = g.next_float();
        for (int a = 0; a < 3; ++a) weight[3 * i + a] = 0.2f + g.next_float();
        for (int a = 0; a < 3; ++a) ipix[3 * i + a] = 0.5f + g.next_float();
        keys[i] = nrrs::root_path_key(i, 0);
    }
    GpuStage gpu(0);
    gpu.set_weights(nets);
    nrrs::RateControl rc;
    const nrrs::Strategy strat{variant == 1 ? nrrs::StrategyKind::AidNrrs : nrrs::StrategyKind::Nrrs, 1.0f};
    const uint32_t depth = 2, n_pixels = n, capacity = nrrs_queue_capacity_for(n_pixels);

    // ---- the adapter call, replacing wavefront.cpp:363-425 ----
    nrrs_vertex_soa v{p01.data(), wo01.data(), rough.data(), weight.data(), ipix.data(), keys.data(), nullptr, nullptr};
    nrrs_stage_params p{};
    p.depth = depth;
    p.n_pixels = n_pixels;
    p.capacity = capacity;
    p.strategy = {static_cast<int32_t>(strat.kind), strat.fixed_value};
    p.gain = rc.gain();
    p.eps_div = 0.0f;
    p.seed = 0;
    std::vector<float> q_norm(n), q_real(n), q_orig(n), u(n);
    std::vector<int32_t> counts(n);
    std::vector<uint32_t> offsets(n), slots(2ull * capacity);
    std::vector<uint8_t> decided(n);
    nrrs_stage_out o{q_norm.data(), q_real.data(), slots.data(), counts.data(), offsets.data(),
                     decided.data(), q_orig.data(), u.data()};
    nrrs_stage_result r{};
    gpu.check(nrrs_gpu_rrs_stage_host(gpu.ctx, &v, n, &p, &o, &r));
    if (r.dropped > 0)
        rc.note_overflow();  // :407-411

    // ---- the reference's own functions on the same inputs ----
    double worst = 0.0;
    for (uint32_t i = 0; i < n; ++i) {
        const nrrs::Vec3f pp(p01[3 * i], p01[3 * i + 1], p01[3 * i + 2]);
        const nrrs::Vec2f wo(wo01[2 * i], wo01[2 * i + 1]);
        const nrrs::Vec3f tx(weight[3 * i], weight[3 * i + 1], weight[3 * i + 2]);
        const nrrs::Vec3f ip(ipix[3 * i], ipix[3 * i + 1], ipix[3 * i + 2]);
        const float qr = nets.predict_q(pp, wo, rough[i], tx, ip);
        worst = std::max(worst, (double)std::fabs(q_orig[i] - qr) / std::max((double)std::fabs(qr), 1e-6));
    }
    EXPECT(worst <= 1e-3, "predict_q vs GPU q_orig: max rel err %.3e", worst);
    std::vector<float> qn = q_orig;
    const double F = nrrs::normalize_factors(qn, n_pixels);  // sequential double sum (rrs.cpp:9-14)
    EXPECT((float)F == (float)r.f_norm, "float(F): reference %.9g, GPU %.9g", F, r.f_norm);
    std::vector<float> qreal(n);
    for (uint32_t i = 0; i < n; ++i) {
        EXPECT(qn[i] == q_norm[i], "q_norm[%u]", i);
        qreal[i] = qn[i] * rc.gain();  // q_real = q * gain (wavefront.cpp:396), before any overflow update
        EXPECT(qreal[i] == q_real[i] || r.dropped > 0, "q_real[%u]", i);
    }
    std::vector<int> k(n);
    const uint64_t total = nrrs::realize_counts(qreal, u, k);  // the reference chain end to end
    EXPECT(total == r.total, "total: reference %llu, GPU %llu", (unsigned long long)total,
           (unsigned long long)r.total);
    uint64_t cum = 0;
    for (uint32_t i = 0; i < n; ++i) {
        EXPECT(k[i] == counts[i], "count[%u]: reference %d, GPU %d", i, k[i], counts[i]);
        EXPECT(offsets[i] == (uint32_t)std::min<uint64_t>(cum, capacity), "offset[%u]", i);  // :148
        cum += (uint64_t)k[i];
        if (failures > 20)
            break;
    }
    const uint64_t spawned = std::min<uint64_t>(cum, capacity);
    EXPECT(spawned == r.spawned, "spawned");
    for (uint64_t s = 0, j = 0, c = 0; s < spawned && failures <= 20; ++s) {  // slot layout (:421-425)
        while (c >= (uint64_t)k[j]) {
            ++j;
            c = 0;
        }
        EXPECT(slots[2 * s] == j && slots[2 * s + 1] == c, "slot %llu", (unsigned long long)s);
        ++c;
    }
    std::printf("{\"variant\": %d, \"n\": %u, \"max_rel_err_q\": %.3e, \"f_norm\": %.17g, \"spawned\": %u, "
                "\"failures\": %d}\n", variant, n, worst, r.f_norm, r.spawned, failures);
    return failures ? 1 : 0;
}
