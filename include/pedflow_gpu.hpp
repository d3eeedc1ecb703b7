// pedflow_gpu.hpp — header-only C++ shim over the C-ABI (pf_gpu.h) that
// re-exposes the reference's step-engine surface for drop-in use:
//
//   reference (/root/reference/proj)            this shim
//   pedflow::StepEngine(EngineOptions)           pedflow::gpu::StepEngine(Options)
//     inc/engine.hpp:48-66
//   StepReport StepEngine::step(SimState&)       StepReport step(SimState&)
//     src/engine.cpp:53-62
//   (none)                                      step_n(SimState&, n, StepReport*) — batched fast path
//   new_environment(cfg, seed)                   pedflow::gpu::new_environment(Options, seed)
//     src/state.cpp:54-75
//
// SimState here holds the reference planes (occupancy, index, agents,
// pheromone) as std::vectors with the reference's layout; AgentRecord and
// StepReport are byte-identical to the reference's, so a maintainer can copy a
// pedflow::SimState into it with memcpy. Errors become exceptions of the same
// classes as the reference: ConfigError (std::runtime_error) and
// std::logic_error("state corrupt: ...").
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "pf_gpu.h"

namespace pedflow::gpu {

struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == PF_OK) return;
    const std::string msg = pf_last_error();
    if (rc == PF_ERR_CONFIG) throw ConfigError(msg);
    if (rc == PF_ERR_STATE) throw std::logic_error(msg);
    throw std::runtime_error("pedflow-b200: " + msg);
}

using StepReport = pf_step_report;
using AgentRecord = pf_agent;

struct Options : pf_config {
    Options() : pf_config{} {
        width = 480;
        height = 480;
        agents_per_side = 1280;
        model = PF_MODEL_ACO;
        seed = 42;
        d0 = 2.0;
        sel_mu = 1.0;
        sel_sigma = 0.5;
        alpha = 1.0;
        beta = 2.0;
        rho = 0.05;
        tau0 = 0.1;
        q = 1.0;
        replicas = 1;
        row_begin = row_end = 0;
        device = 0;
        kernel = PF_KERNEL_FUSED;
    }
};

struct SimState {
    int width = 0, height = 0, model = PF_MODEL_LEM;
    std::vector<uint8_t> occupancy;
    std::vector<uint32_t> index;
    std::vector<AgentRecord> agents;
    std::vector<double> pheromone_top, pheromone_bottom;
    std::vector<double> scores;  // CandidateScores::score by agent id, [n][8] (filled by the phase methods)
    uint32_t step = 0;
};

inline SimState new_environment(const Options& o, uint64_t seed) {
    SimState s;
    s.width = o.width;
    s.height = o.height;
    s.model = o.model;
    const size_t cells = size_t(o.width) * size_t(o.height);
    s.occupancy.assign(cells, 0);
    s.index.assign(cells, 0);
    s.agents.assign(2 * size_t(o.agents_per_side > 0 ? o.agents_per_side : 0), AgentRecord{});
    if (o.model == PF_MODEL_ACO) {
        s.pheromone_top.assign(cells, 0.0);
        s.pheromone_bottom.assign(cells, 0.0);
    }
    check(pf_new_environment(&o, seed, s.occupancy.data(), s.index.data(), s.agents.data(),
                             s.pheromone_top.empty() ? nullptr : s.pheromone_top.data(),
                             s.pheromone_bottom.empty() ? nullptr : s.pheromone_bottom.data()));
    return s;
}

class StepEngine {
  public:
    explicit StepEngine(const Options& o) : opt_(o) { check(pf_create(&opt_, &ctx_)); }
    ~StepEngine() { pf_destroy(ctx_); }
    StepEngine(const StepEngine&) = delete;
    StepEngine& operator=(const StepEngine&) = delete;

    // Drop-in: one synchronous step of `s` (upload, step, download).
    StepReport step(SimState& s) {
        StepReport r{};
        step_n(s, 1, &r);
        return r;
    }

    // Batched: n steps with one upload and one download; reports may be null.
    void step_n(SimState& s, uint32_t n, StepReport* reports) {
        upload(s);
        check(pf_step(ctx_, n, reports));
        download(s);
    }

    void upload(const SimState& s) {
        check(pf_load_state(ctx_, 0, s.occupancy.data(), s.index.data(), s.agents.data(), uint32_t(s.agents.size()),
                            s.pheromone_top.empty() ? nullptr : s.pheromone_top.data(),
                            s.pheromone_bottom.empty() ? nullptr : s.pheromone_bottom.data(), s.step));
    }
    void download(SimState& s) {
        check(pf_store_state(ctx_, 0, s.occupancy.data(), s.index.data(), s.agents.data(), uint32_t(s.agents.size()),
                             s.pheromone_top.empty() ? nullptr : s.pheromone_top.data(),
                             s.pheromone_bottom.empty() ? nullptr : s.pheromone_bottom.data(), &s.step));
    }

    // Phase-level stepping (StepEngine::score_phase .. reset_phase,
    // src/engine.cpp:64-193); needs Options::kernel = PF_KERNEL_PIPELINE.
    // score_phase uploads `s`; the later phases of the same step continue on
    // the device (do not modify `s` in between); each downloads the result,
    // so s.agents' futures and s.scores read as the reference's do.
    void score_phase(SimState& s) {
        upload(s);
        phase(s, PF_PHASE_SCORE, nullptr);
    }
    void intention_phase(SimState& s) { phase(s, PF_PHASE_INTENTION, nullptr); }
    StepReport movement_phase(SimState& s) {
        StepReport r{};
        phase(s, PF_PHASE_MOVEMENT, &r);
        return r;
    }
    void reset_phase(SimState& s) { phase(s, PF_PHASE_RESET, nullptr); }

    const Options& options() const { return opt_; }
    pf_ctx* handle() { return ctx_; }

  private:
    void phase(SimState& s, int32_t ph, StepReport* r) {
        check(pf_phase(ctx_, ph, r));
        download(s);
        s.scores.resize(s.agents.size() * 8);
        check(pf_store_scores(ctx_, 0, s.scores.data(), nullptr, uint32_t(s.agents.size())));
    }

    Options opt_;
    pf_ctx* ctx_ = nullptr;
};

}  // namespace pedflow::gpu
