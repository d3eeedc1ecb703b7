// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/).
// Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline
// legs may load the resulting library. It exposes exactly the reference calls
// the hot path sits behind:
//   new_environment        (inc/state.hpp:37, src/state.cpp:54-75)
//   EngineOptions::from_config (src/engine.cpp:35-46)
//   StepEngine::step       (inc/engine.hpp:51, src/engine.cpp:53-62)
// The step loop is timed on its own (run_scenario's clock includes setup,
// src/engine.cpp:198), which is what SURVEY.md §8(d) asks for.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "pedflow/config.hpp"
#include "pedflow/engine.hpp"
#include "pedflow/state.hpp"

namespace {

thread_local std::string g_err;

struct RefHandle {
    pedflow::ScenarioConfig cfg;
    pedflow::SimState state;
    std::unique_ptr<pedflow::StepEngine> engine;
};

}  // namespace

extern "C" {

// Mirrors the numeric part of ScenarioConfig (inc/config.hpp:20-58).
struct ref_cfg {
    int32_t width, height, agents_per_side, model;  // model: 0 LEM, 1 ACO
    uint64_t seed;
    double d0, sel_mu, sel_sigma, alpha, beta, rho, tau0, q;
};

const char* ref_last_error() { return g_err.c_str(); }

// threads <= 0: Sequential executor; otherwise Parallel with that many threads.
void* ref_create(const ref_cfg* c, int threads) {
    try {
        auto h = std::make_unique<RefHandle>();
        pedflow::ScenarioConfig& cfg = h->cfg;
        cfg.width = c->width;
        cfg.height = c->height;
        cfg.agents_per_side = c->agents_per_side;
        cfg.model = c->model == 0 ? pedflow::Model::Lem : pedflow::Model::Aco;
        cfg.seed = c->seed;
        cfg.d0 = c->d0;
        cfg.sel_mu = c->sel_mu;
        cfg.sel_sigma = c->sel_sigma;
        cfg.alpha = c->alpha;
        cfg.beta = c->beta;
        cfg.rho = c->rho;
        cfg.tau0 = c->tau0;
        cfg.q = c->q;
        cfg.executor = threads > 0 ? pedflow::ExecutorKind::Parallel : pedflow::ExecutorKind::Sequential;
        cfg.threads = threads > 0 ? threads : 0;
        pedflow::validate(cfg);
        h->state = pedflow::new_environment(cfg, c->seed);
        pedflow::EngineOptions opt = pedflow::EngineOptions::from_config(cfg, c->seed);
        h->engine = std::make_unique<pedflow::StepEngine>(std::move(opt));
        return h.release();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_destroy(void* p) { delete static_cast<RefHandle*>(p); }

// Switches the executor of an existing handle (threads <= 0: Sequential,
// else Parallel with that many threads) by rebuilding its StepEngine from the
// config (EngineOptions::from_config, src/engine.cpp:35-46); the SimState and
// its step counter are kept, so Sequential and Parallel can be timed on one
// placement (the reference's `bench` compares the two executors the same way,
// tools/pedflow.cpp:191-225).
int ref_set_executor(void* p, int threads) {
    try {
        auto* h = static_cast<RefHandle*>(p);
        h->cfg.executor = threads > 0 ? pedflow::ExecutorKind::Parallel : pedflow::ExecutorKind::Sequential;
        h->cfg.threads = threads > 0 ? threads : 0;
        pedflow::EngineOptions opt = pedflow::EngineOptions::from_config(h->cfg, h->cfg.seed);
        h->engine = std::make_unique<pedflow::StepEngine>(std::move(opt));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

// Runs n steps; reports is n*4 u32 (StepReport layout) or null. *seconds gets
// the wall time of the step loop alone.
int ref_step(void* p, uint32_t n, uint32_t* reports, double* seconds) {
    try {
        auto* h = static_cast<RefHandle*>(p);
        const auto t0 = std::chrono::steady_clock::now();
        for (uint32_t i = 0; i < n; ++i) {
            const pedflow::StepReport r = h->engine->step(h->state);
            if (reports) {
                reports[4 * i + 0] = r.step;
                reports[4 * i + 1] = r.moved;
                reports[4 * i + 2] = r.newly_crossed_top;
                reports[4 * i + 3] = r.newly_crossed_bottom;
            }
        }
        if (seconds)
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

uint32_t ref_agent_count(void* p) { return uint32_t(static_cast<RefHandle*>(p)->state.agents.size()); }

// Copies the state out. agents receives raw AgentRecord bytes (40 B each).
// tau_* may be null (LEM).
int ref_export(void* p, uint8_t* occ, uint32_t* index, void* agents, double* tau_top,
               double* tau_bot, uint32_t* step) {
    auto* h = static_cast<RefHandle*>(p);
    const pedflow::SimState& s = h->state;
    const size_t cells = size_t(s.width) * size_t(s.height);
    if (occ) std::memcpy(occ, s.occupancy.data().data(), cells);
    if (index) std::memcpy(index, s.index.data().data(), cells * 4);
    if (agents) std::memcpy(agents, s.agents.data(), s.agents.size() * sizeof(pedflow::AgentRecord));
    if (tau_top && !s.pheromone.empty())
        std::memcpy(tau_top, s.pheromone.top.data().data(), cells * 8);
    if (tau_bot && !s.pheromone.empty())
        std::memcpy(tau_bot, s.pheromone.bottom.data().data(), cells * 8);
    if (step) *step = s.step;
    return 0;
}

uint32_t ref_agent_record_size() { return uint32_t(sizeof(pedflow::AgentRecord)); }

// Direct access to the reference RNG for known-answer checks (src/rng.cpp:43-59).
uint64_t ref_random_bits(uint64_t seed, uint32_t step, uint32_t phase, uint64_t entity,
                         uint32_t counter) {
    return pedflow::random_bits(
        pedflow::RngKey{seed, step, pedflow::Phase(phase), entity, counter});
}
double ref_normal(uint64_t seed, uint32_t step, uint32_t phase, uint64_t entity, uint32_t counter,
                  double mu, double sigma) {
    return pedflow::normal(pedflow::RngKey{seed, step, pedflow::Phase(phase), entity, counter},
                           mu, sigma);
}
double ref_inverse_normal_cdf(double p) { return pedflow::inverse_normal_cdf(p); }

}  // extern "C"
