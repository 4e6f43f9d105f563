// ref_cli.cpp — extern "C" harness over the REAL reference's config parser,
// record writer and CLI command bodies (TEST INFRASTRUCTURE ONLY).
//
// The reference CLI (src/cli.cpp) needs CLI11, which is absent here, so its
// command bodies are restated below on top of the reference's own
// load_config / make_*_spec / observe_* / run_chain / optimize_forcing /
// RecordWriter (compiled in place by oracle/Makefile).  tests/golden/
// make_golden.py uses them to write the golden CLI outputs that
// paper_1808_10580_b200.cli is checked against, and tests/test_config.py
// compares paper_1808_10580_b200.config's diagnostics with parse_config's.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "scalarmc/config.hpp"
#include "scalarmc/forward_ad.hpp"
#include "scalarmc/forward_bvp.hpp"
#include "scalarmc/inference.hpp"
#include "scalarmc/io.hpp"
#include "scalarmc/optimize.hpp"

using namespace scalarmc;

namespace {

void copy_out(const std::string& s, char* buf, int cap) {
    if (!buf || cap <= 0) return;
    std::snprintf(buf, static_cast<size_t>(cap), "%s", s.c_str());
}

// 0 ok, 1 ConfigError, 2 invalid_argument, 3 out_of_range, 4 other exception
template <class F>
int classify(F&& f, char* msg, int cap) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        copy_out(e.what(), msg, cap);
        return 1;
    } catch (const std::invalid_argument& e) {
        copy_out(e.what(), msg, cap);
        return 2;
    } catch (const std::out_of_range& e) {
        copy_out(e.what(), msg, cap);
        return 3;
    } catch (const std::exception& e) {
        copy_out(e.what(), msg, cap);
        return 4;
    }
}

std::ofstream open_out(const std::string& path) {
    const auto parent = std::filesystem::path(path).parent_path();
    if (!parent.empty()) std::filesystem::create_directories(parent);
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open output file: " + path);
    return out;
}

}  // namespace

extern "C" {

// parse_config(text, origin) and then, by `stage`: 1 make_ad_spec,
// 2 make_bvp_spec, 3 make_likelihood, 4 make_forcing_control.
int refcli_config_check(const char* text, const char* origin, int stage, char* msg, int cap) {
    return classify(
        [&] {
            const RunConfig cfg = parse_config(text, origin);
            if (stage == 1) (void)make_ad_spec(cfg);
            if (stage == 2) (void)make_bvp_spec(cfg);
            if (stage == 3) (void)make_likelihood(cfg);
            if (stage == 4) (void)make_forcing_control(cfg);
        },
        msg, cap);
}

void refcli_format_double(double v, char* buf, int cap) { copy_out(format_double(v), buf, cap); }

// cmd_forward_ad / cmd_forward_bvp (cli.cpp:63-96) with seed override
// (< 0: the config's seed); workers = all hardware threads.
int refcli_forward(const char* config_path, const char* out_path, const char* fmt, int64_t seed, int bvp, char* msg,
                   int cap) {
    return classify(
        [&] {
            const RunConfig cfg = load_config(config_path);
            const std::uint64_t s = seed >= 0 ? static_cast<std::uint64_t>(seed) : cfg.seed;
            auto out = open_out(out_path);
            if (!bvp) {
                const AdProblemSpec spec = make_ad_spec(cfg);
                const auto est = observe_ad(spec, s, 0);
                RecordWriter w(out, parse_record_format(fmt),
                               {"t", "x1", "x2", "mean", "std_error", "n_particles", "n_failed"});
                for (std::size_t j = 0; j < est.size(); ++j) {
                    const auto& o = spec.observations[j];
                    const std::vector<double> row{o.t,          o.x.x1,           o.x.x2, est[j].mean,
                                                  est[j].std_error, double(est[j].n_particles),
                                                  double(est[j].n_failed)};
                    w.write_row(row);
                }
            } else {
                const BvpProblemSpec spec = make_bvp_spec(cfg);
                const auto est = observe_bvp(spec, s, 0);
                RecordWriter w(out, parse_record_format(fmt),
                               {"x1", "x2", "mean", "std_error", "mean_exit_time", "n_failed"});
                for (std::size_t j = 0; j < est.size(); ++j) {
                    const auto& x = spec.observations[j];
                    const std::vector<double> row{x.x1, x.x2, est[j].mean, est[j].std_error, est[j].aux_mean,
                                                  double(est[j].n_failed)};
                    w.write_row(row);
                }
            }
        },
        msg, cap);
}

// cmd_sample (cli.cpp:140-199): files under out_dir, stdout text into `text`.
int refcli_sample(const char* config_path, const char* out_dir, const char* fmt_name, int64_t seed,
                  int64_t steps_override, double beta_override, char* text, int text_cap, char* msg, int cap) {
    return classify(
        [&] {
            const RunConfig cfg = load_config(config_path);
            if (!cfg.prior) throw ConfigError("prior", "section required by `sample`");
            const PriorSpec prior = *cfg.prior;
            LikelihoodSpec likelihood = make_likelihood(cfg);
            likelihood.workers = 0;
            McmcSection mc = cfg.mcmc.value_or(McmcSection{});
            if (steps_override >= 0) mc.steps = steps_override;
            if (beta_override > 0.0) mc.beta = beta_override;
            const std::uint64_t s = seed >= 0 ? static_cast<std::uint64_t>(seed) : cfg.seed;
            const ChainConfig cc{mc.steps, mc.beta, mc.burn_in, mc.thin, s};
            const ChainResult r = run_chain(cc, prior, &likelihood);
            std::filesystem::create_directories(out_dir);
            const std::string fmt = fmt_name;
            const auto f = parse_record_format(fmt);
            const int dim = prior.dimension();
            std::vector<std::string> cols{"iteration", "phi"}, ucols;
            for (int c = 0; c < dim; ++c) ucols.push_back("u" + std::to_string(c));
            cols.insert(cols.end(), ucols.begin(), ucols.end());
            {
                auto out = open_out(std::string(out_dir) + "/archive." + fmt);
                RecordWriter w(out, f, cols);
                for (std::size_t i = 0; i < r.samples.size(); ++i) {
                    const auto it = cc.burn_in + std::int64_t(i) * cc.thin + 1;
                    std::vector<double> row{double(it), r.phi_trace[std::size_t(it - 1)]};
                    row.insert(row.end(), r.samples[i].begin(), r.samples[i].end());
                    w.write_row(row);
                }
            }
            {
                auto out = open_out(std::string(out_dir) + "/map." + fmt);
                RecordWriter w(out, f, ucols);
                w.write_row(r.map_u);
            }
            {
                auto out = open_out(std::string(out_dir) + "/summary." + fmt);
                RecordWriter w(out, f,
                               {"steps", "acceptance_rate", "map_objective", "final_phi", "flagged_failures",
                                "samples"});
                const std::vector<double> row{double(mc.steps), r.acceptance_rate, r.map_objective,
                                              r.final_state.phi, double(r.final_state.flagged_failures),
                                              double(r.samples.size())};
                w.write_row(row);
            }
            std::ostringstream o;
            o << "acceptance_rate " << format_double(r.acceptance_rate) << "\n"
              << "map_objective " << format_double(r.map_objective) << "\n"
              << "samples " << r.samples.size() << "\n";
            copy_out(o.str(), text, text_cap);
        },
        msg, cap);
}

// cmd_optimize (cli.cpp:201-228).
int refcli_optimize(const char* config_path, const char* out_path, const char* fmt, int64_t seed, char* text,
                    int text_cap, char* msg, int cap) {
    return classify(
        [&] {
            const RunConfig cfg = load_config(config_path);
            const BvpProblemSpec base = make_bvp_spec(cfg);
            const ForcingControl control = make_forcing_control(cfg);
            const std::uint64_t s = seed >= 0 ? static_cast<std::uint64_t>(seed) : cfg.seed;
            const auto r = optimize_forcing(control, base, cfg.optimize->options, s, 0);
            auto out = open_out(out_path);
            std::vector<std::string> cols{"iteration", "best_cost"};
            for (std::size_t c = 0; c < control.centers.size(); ++c) cols.push_back("f" + std::to_string(c));
            RecordWriter w(out, parse_record_format(fmt), cols);
            for (const auto& e : r.trace) {
                std::vector<double> row{double(e.iteration), e.best_value};
                row.insert(row.end(), e.best_point.begin(), e.best_point.end());
                w.write_row(row);
            }
            std::ostringstream o;
            o << "best_cost " << format_double(r.min_value) << "\n"
              << "iterations " << r.iterations << " (" << r.stop_reason << ")\n"
              << "amplitudes";
            for (double v : r.argmin) o << ' ' << format_double(v);
            o << "\n";
            copy_out(o.str(), text, text_cap);
        },
        msg, cap);
}

}  // extern "C"
