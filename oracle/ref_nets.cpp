// Drives the reference's own networks.cpp / mlp.cpp / hashgrid.cpp (compiled unmodified from
// /root/reference against oracle/eigen_shim) through a C ABI, for the golden fixtures of
// tests/golden/make_ref_golden.py.  Test infrastructure only: built into oracle/_ref/ (git-ignored)
// by `make -C oracle ref` when the reference tree is present.
#include "nrrs/networks.hpp"

#include <cstdio>
#include <exception>

extern "C" {

// Loads a NRRSCK01 checkpoint with the reference's NeuralRrs::load_checkpoint (networks.cpp:641-705)
// and evaluates predict_q (networks.cpp:266-281) and predict_stats (:252-264) on n vertices.
int ref_predict(const char *ckpt, int variant, int levels, int features, int base_resolution,
                int log2_table_size, size_t n, const float *p01, const float *wo01, const float *roughness,
                const float *t_x, const float *i_pixel, float *q_out, float *stats_out) {
    try {
        nrrs::NeuralRrsConfig cfg;
        cfg.variant = variant == 1 ? nrrs::RrsVariant::Aid : nrrs::RrsVariant::Nrrs;
        cfg.grid.levels = levels;
        cfg.grid.features = features;
        cfg.grid.base_resolution = base_resolution;
        cfg.grid.log2_table_size = log2_table_size;
        nrrs::NeuralRrs nets(cfg);
        nets.load_checkpoint(ckpt);
        for (size_t i = 0; i < n; ++i) {
            const nrrs::Vec3f p(p01[3 * i], p01[3 * i + 1], p01[3 * i + 2]);
            const nrrs::Vec2f wo(wo01[2 * i], wo01[2 * i + 1]);
            const nrrs::Vec3f tx(t_x[3 * i], t_x[3 * i + 1], t_x[3 * i + 2]);
            const nrrs::Vec3f ip(i_pixel[3 * i], i_pixel[3 * i + 1], i_pixel[3 * i + 2]);
            q_out[i] = nets.predict_q(p, wo, roughness[i], tx, ip);
            if (stats_out) {
                const nrrs::RadianceStats st = nets.predict_stats(p, wo, roughness[i]);
                for (int k = 0; k < 3; ++k) {
                    stats_out[6 * i + k] = st.mean[k];
                    stats_out[6 * i + 3 + k] = st.second_moment[k];
                }
            }
        }
        return 0;
    } catch (const std::exception &e) {
        std::fprintf(stderr, "ref_predict: %s\n", e.what());
        return -1;
    }
}
}
