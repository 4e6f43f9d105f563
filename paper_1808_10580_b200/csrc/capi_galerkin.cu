// capi_galerkin.cu — C ABI of the spectral Galerkin reference solver
// (src/galerkin.cpp).
#include "capi_internal.h"

using namespace smc;
using namespace smc::capi;

namespace {
// check_galerkin_inputs (galerkin.cpp:144-149): the spec's own validation
// (isotropic diffusion is the only kind the ABI carries).
PreparedVelocity galerkin_check_inputs(const smc_ad_problem& p) {
    PreparedVelocity v = prepare_velocity(p.velocity);
    check_kappa(p.kappa);
    check_scalar(p.initial_condition);
    ad_validate(p);
    return v;
}
}  // namespace

extern "C" {

// ---- spectral Galerkin reference solver (src/galerkin.cpp) ----------------


int64_t smc_galerkin_n_basis(const smc_galerkin_basis* basis) {
    try {
        return galerkin_modes(*basis).size();
    } catch (...) {
        return -1;
    }
}

smc_status smc_galerkin_modes(const smc_galerkin_basis* basis, int32_t* modes) {
    return guarded(__func__, [&] {
        const GalerkinModes m = galerkin_modes(*basis);
        for (int64_t i = 0; i < m.size(); ++i) {
            modes[2 * i] = m.k1[static_cast<size_t>(i)];
            modes[2 * i + 1] = m.k2[static_cast<size_t>(i)];
        }
    });
}

smc_status smc_galerkin_spectral_radius(smc_ctx*, const smc_ad_problem* prob, const smc_galerkin_basis* basis,
                                        double* out) {
    return guarded(__func__, [&] {
        const PreparedVelocity v = galerkin_check_inputs(*prob);
        const GalerkinModes m = galerkin_modes(*basis);
        *out = galerkin_radius(galerkin_assemble(prob->kappa, v, m), m.size());
    });
}

smc_status smc_galerkin_solve_ad(smc_ctx* ctx, const smc_ad_problem* prob, const smc_galerkin_basis* basis,
                                 double dt_ref, smc_galerkin_result* out) {
    return guarded(__func__, [&] {
        CK(cudaSetDevice(ctx->device));
        const smc_ad_problem& p = *prob;
        const PreparedVelocity v = galerkin_check_inputs(p);
        if (!(dt_ref > 0.0)) raise(SMC_EINVAL, "galerkin_solve_ad: dt_ref must be positive");
        const GalerkinModes m = galerkin_modes(*basis);
        const int64_t nb = m.size();
        cudaStream_t s = ctx->stream;
        double* dA = ctx->gal_A.get<double>(static_cast<size_t>(2 * nb * nb));
        double* th[2] = {ctx->gal_t0.get<double>(static_cast<size_t>(2 * nb)),
                         ctx->gal_t1.get<double>(static_cast<size_t>(2 * nb))};
        int* dk1 = ctx->gal_k1.get<int>(static_cast<size_t>(nb));
        int* dk2 = ctx->gal_k2.get<int>(static_cast<size_t>(nb));
        double* dobs = ctx->gal_obs.get<double>(static_cast<size_t>(std::max<int64_t>(p.n_obs, 1)));
        CK(cudaMemcpyAsync(dk1, m.k1.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dk2, m.k2.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, s));
        // A assembled on the device (bit-identical to the host restatement of
        // galerkin.cpp:108-142), then the explicit-Euler stability estimate
        // (galerkin.cpp:170-177)
        const VhatGrid vg = galerkin_vhat_grid(v);
        const size_t cells = vg.present.size();
        double* dvh = ctx->gal_grid.get<double>(4 * cells + (cells + 7) / 8 + 1);
        auto* dpres = reinterpret_cast<unsigned char*>(dvh + 4 * cells);
        auto* dradius = ctx->tmp_a.get<unsigned long long>(1);
        CK(cudaMemcpyAsync(dvh, vg.c.data(), sizeof(double) * 4 * cells, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dpres, vg.present.data(), cells, cudaMemcpyHostToDevice, s));
        CK(launch_galerkin_assemble(dvh, dpres, vg.K, dk1, dk2, nb, p.kappa, v.is_constant ? 1 : 0, v.c1, v.c2, dA,
                                    dradius, s));
        count_launches(ctx, 2);
        unsigned long long rbits = 0;
        CK(cudaMemcpyAsync(&rbits, dradius, sizeof(rbits), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double radius;
        std::memcpy(&radius, &rbits, sizeof(radius));
        if (radius * dt_ref >= 2.0) {
            std::ostringstream msg;
            msg << "galerkin_solve_ad: dt_ref " << dt_ref << " violates the stability estimate; suggest dt_ref <= "
                << 1.8 / radius;
            raise(SMC_ERUNTIME, msg.str());
        }
        // projection of theta_0 (galerkin.cpp:43-101)
        std::vector<double> theta0;
        if (galerkin_project_exact(p.initial_condition, m, theta0)) {
            CK(cudaMemcpyAsync(th[0], theta0.data(), sizeof(double) * 2 * nb, cudaMemcpyHostToDevice, s));
        } else {
            Image im;
            const ScalarRef ref = add_scalar(im, p.initial_condition);
            unsigned char* base = ctx->upload(im);
            const int n = std::max(128, 4 * (m.max_abs + 1));
            CK(launch_galerkin_quadrature(patch(ref, base), dk1, dk2, nb, n, th[0], s));
            count_launches(ctx, 1);
        }
        // the step schedule: once through the sorted observation times, shortening
        // the last step of each segment to land on t_j (galerkin.cpp:181-221)
        std::vector<int64_t> order(static_cast<size_t>(p.n_obs));
        for (int64_t i = 0; i < p.n_obs; ++i) order[static_cast<size_t>(i)] = i;
        std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return p.obs_t[a] < p.obs_t[b]; });
        constexpr int kGroup = 16;  // even: a group returns to the buffer it started from
        cudaGraphExec_t group[2] = {nullptr, nullptr};
        struct GraphFree {
            cudaGraphExec_t* g;
            ~GraphFree() {
                for (int i = 0; i < 2; ++i)
                    if (g[i]) cudaGraphExecDestroy(g[i]);
            }
        } graph_free{group};
        auto group_exec = [&](int cur) {
            if (!group[cur]) {
                cudaGraph_t graph = nullptr;
                CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
                cudaError_t e = cudaSuccess;
                for (int k = 0; k < kGroup && e == cudaSuccess; ++k)
                    e = launch_galerkin_step(dA, th[(cur + k) & 1], th[(cur + k + 1) & 1], nb, dt_ref, s);
                const cudaError_t e2 = cudaStreamEndCapture(s, &graph);
                CK(e);
                CK(e2);
                const cudaError_t e3 = cudaGraphInstantiate(&group[cur], graph, 0);
                cudaGraphDestroy(graph);
                CK(e3);
            }
            return group[cur];
        };
        int cur = 0;
        double t = 0.0;
        int64_t steps = 0;
        const bool use_graph = s != nullptr;
        for (const int64_t oi : order) {
            const double target = p.obs_t[oi];
            int64_t run = 0;  // pending full steps of dt_ref
            auto flush = [&] {
                for (; use_graph && run >= kGroup; run -= kGroup) {
                    CK(cudaGraphLaunch(group_exec(cur), s));
                    count_launches(ctx, kGroup);
                }
                for (; run > 0; --run, cur ^= 1) {
                    CK(launch_galerkin_step(dA, th[cur], th[cur ^ 1], nb, dt_ref, s));
                    count_launches(ctx, 1);
                }
            };
            while (t < target - 1e-15) {
                const double dt = std::min(dt_ref, target - t);
                if (dt == dt_ref) {
                    ++run;
                } else {
                    flush();
                    CK(launch_galerkin_step(dA, th[cur], th[cur ^ 1], nb, dt, s));
                    count_launches(ctx, 1);
                    cur ^= 1;
                }
                t += dt;
                ++steps;
            }
            flush();
            CK(launch_galerkin_observe(th[cur], dk1, dk2, nb, p.obs_x[2 * oi], p.obs_x[2 * oi + 1], dobs + oi, s));
            count_launches(ctx, 1);
            if (out->coefficients_at_observations)
                CK(cudaMemcpyAsync(out->coefficients_at_observations + oi * 2 * nb, th[cur], sizeof(double) * 2 * nb,
                                   cudaMemcpyDeviceToHost, s));
        }
        CK(cudaMemcpyAsync(out->observation_values, dobs, sizeof(double) * p.n_obs, cudaMemcpyDeviceToHost, s));
        if (out->final_coefficients)
            CK(cudaMemcpyAsync(out->final_coefficients, th[cur], sizeof(double) * 2 * nb, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        out->dt_used = dt_ref;
        out->steps = steps;
    });
}

smc_status smc_galerkin_field_grid(smc_ctx* ctx, const smc_galerkin_basis* basis, const double* coefficients,
                                   int32_t n, double* grid) {
    return guarded(__func__, [&] {
        CK(cudaSetDevice(ctx->device));
        if (n < 2) raise(SMC_EINVAL, "galerkin_field_grid: n must be >= 2");
        const GalerkinModes m = galerkin_modes(*basis);
        const int64_t nb = m.size();
        cudaStream_t s = ctx->stream;
        double* dc = ctx->gal_t0.get<double>(static_cast<size_t>(2 * nb));
        int* dk1 = ctx->gal_k1.get<int>(static_cast<size_t>(nb));
        int* dk2 = ctx->gal_k2.get<int>(static_cast<size_t>(nb));
        double* dg = ctx->gal_grid.get<double>(static_cast<size_t>(n) * n);
        CK(cudaMemcpyAsync(dc, coefficients, sizeof(double) * 2 * nb, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dk1, m.k1.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dk2, m.k2.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, s));
        CK(launch_galerkin_field_grid(dc, dk1, dk2, nb, n, dg, s));
        count_launches(ctx, 1);
        CK(cudaMemcpyAsync(grid, dg, sizeof(double) * n * n, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
