// pedflow_gpu.hpp — header-only C++ shim over the C-ABI (pf_gpu.h) that
// re-exposes the reference's step-engine surface for drop-in use:
//
//   reference (/root/reference/proj)            this shim
//   pedflow::StepEngine(EngineOptions)           pedflow::gpu::StepEngine(Options)
//     inc/engine.hpp:48-66
//   StepReport StepEngine::step(SimState&)       StepReport step(SimState&) — lazy: the state stays
//     src/engine.cpp:53-62                         on the device between calls (SimState::sync())
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

#include <atomic>
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

class StepEngine;

// SimState: the reference planes in the reference layout, plus the lazy-sync
// bookkeeping of SURVEY.md §8(b) ("syncing state lazily"). A StepEngine keeps
// the state device-resident across step() calls: it uploads only when the
// state is not the one it holds or the host planes changed, and it does not
// download after a step. The host planes are refreshed by sync() (also done
// by copying the state, by the phase methods, by stepping it on another
// engine, and by the holding engine's destructor). `step` is always current.
// After modifying planes on the host call mark_dirty() (sync() first if the
// state was being stepped) so the next step re-uploads.
struct SimState {
    int width = 0, height = 0, model = PF_MODEL_LEM;
    std::vector<uint8_t> occupancy;
    std::vector<uint32_t> index;
    std::vector<AgentRecord> agents;
    std::vector<double> pheromone_top, pheromone_bottom;
    std::vector<double> scores;  // CandidateScores::score by agent id, [n][8] (filled by the phase methods)
    uint32_t step = 0;

    SimState() = default;
    SimState(const SimState& o);             // snapshot (syncs `o` first)
    SimState(SimState&& o) noexcept;         // takes over o's residency
    SimState& operator=(const SimState& o);
    SimState& operator=(SimState&& o) noexcept;
    ~SimState();

    void sync() const;                       // host planes := newest copy
    void mark_dirty() { detach(); ++version_; }
    bool device_newer() const { return holder_ != nullptr; }

  private:
    friend class StepEngine;
    void detach();  // forget the device copy without downloading
    void copy_planes(const SimState& o) {
        width = o.width, height = o.height, model = o.model;
        occupancy = o.occupancy, index = o.index, agents = o.agents;
        pheromone_top = o.pheromone_top, pheromone_bottom = o.pheromone_bottom;
        scores = o.scores, step = o.step;
    }
    void move_planes(SimState& o) {
        width = o.width, height = o.height, model = o.model;
        occupancy = std::move(o.occupancy), index = std::move(o.index), agents = std::move(o.agents);
        pheromone_top = std::move(o.pheromone_top), pheromone_bottom = std::move(o.pheromone_bottom);
        scores = std::move(o.scores), step = o.step;
    }
    static uint64_t next_token() {
        static std::atomic<uint64_t> t{1};
        return t.fetch_add(1);
    }
    uint64_t token_ = next_token();  // identity that is never reused
    uint64_t version_ = 0;            // bumped whenever the host planes change
    StepEngine* holder_ = nullptr;    // engine whose device copy is newer than the planes
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
    ~StepEngine() {
        if (newer_) {
            try {
                newer_->sync();  // the state outlives its device copy
            } catch (...) {
            }
        }
        pf_destroy(ctx_);
    }
    StepEngine(const StepEngine&) = delete;
    StepEngine& operator=(const StepEngine&) = delete;

    // Drop-in StepEngine::step(SimState&) (src/engine.cpp:53-62): one step,
    // state kept on the device (see SimState). One graph launch plus the
    // 16-byte report read per call.
    StepReport step(SimState& s) {
        StepReport r{};
        step_n(s, 1, &r);
        return r;
    }

    // n steps under one CUDA graph batch; reports may be null. Lazy like step().
    void step_n(SimState& s, uint32_t n, StepReport* reports) {
        attach(s, false);
        check(pf_step(ctx_, n, reports));
        s.step += n;
    }

    // Eager transfer: upload `s` now even if the device copy looks current.
    void upload(SimState& s) { attach(s, true); }

    // Phase-level stepping (StepEngine::score_phase .. reset_phase,
    // src/engine.cpp:64-193); needs Options::kernel = PF_KERNEL_PIPELINE.
    // Each phase continues on the device copy and then downloads, so
    // s.agents' futures and s.scores read as the reference's do.
    void score_phase(SimState& s) { phase(s, PF_PHASE_SCORE, nullptr); }
    void intention_phase(SimState& s) { phase(s, PF_PHASE_INTENTION, nullptr); }
    StepReport movement_phase(SimState& s) {
        StepReport r{};
        phase(s, PF_PHASE_MOVEMENT, &r);
        return r;
    }
    void reset_phase(SimState& s) { phase(s, PF_PHASE_RESET, nullptr); }

    const Options& options() const { return opt_; }
    pf_ctx* handle() { return ctx_; }
    uint64_t uploads() const { return uploads_; }
    uint64_t downloads() const { return downloads_; }

  private:
    friend struct SimState;

    // Make the device hold `s`'s newest planes; afterwards the device copy is
    // the one that advances (s.holder_ == this).
    void attach(SimState& s, bool force) {
        if (s.holder_ == this && !force) return;  // resident and newer on the device
        s.sync();  // newer on another engine (or here, when forced): bring it home first
        if (force || bound_token_ != s.token_ || bound_version_ != s.version_) {
            if (newer_ && newer_ != &s) newer_->sync();  // the other state must not lose its steps
            check(pf_load_state(ctx_, 0, s.occupancy.data(), s.index.data(), s.agents.data(),
                                uint32_t(s.agents.size()), s.pheromone_top.empty() ? nullptr : s.pheromone_top.data(),
                                s.pheromone_bottom.empty() ? nullptr : s.pheromone_bottom.data(), s.step));
            ++uploads_;
            bound_token_ = s.token_;
            bound_version_ = s.version_;
        }
        newer_ = &s;
        s.holder_ = this;
    }
    // Host planes := this engine's device copy (only for the state it holds).
    void download(SimState& s) {
        if (newer_ != &s) throw std::logic_error("pedflow-b200: download of a state this engine does not hold");
        check(pf_store_state(ctx_, 0, s.occupancy.data(), s.index.data(), s.agents.data(), uint32_t(s.agents.size()),
                             s.pheromone_top.empty() ? nullptr : s.pheromone_top.data(),
                             s.pheromone_bottom.empty() ? nullptr : s.pheromone_bottom.data(), &s.step));
        ++downloads_;
        newer_ = nullptr;
        s.holder_ = nullptr;
        ++s.version_;  // other engines' copies are stale now; ours equals the planes
        bound_token_ = s.token_;
        bound_version_ = s.version_;
    }
    void phase(SimState& s, int32_t ph, StepReport* r) {
        attach(s, false);
        check(pf_phase(ctx_, ph, r));
        download(s);
        s.scores.resize(s.agents.size() * 8);
        check(pf_store_scores(ctx_, 0, s.scores.data(), nullptr, uint32_t(s.agents.size())));
    }
    // SimState bookkeeping hooks (destruction, move, overwrite of a held state).
    void forget(const SimState* s) {
        if (newer_ == s) newer_ = nullptr, bound_token_ = 0;
    }
    void moved(const SimState* from, SimState* to) {
        if (newer_ == from) newer_ = to;
    }

    Options opt_;
    pf_ctx* ctx_ = nullptr;
    SimState* newer_ = nullptr;  // the state whose newest planes live on this device (holder_ == this)
    uint64_t bound_token_ = 0, bound_version_ = 0;  // the (state, version) the device copy started from
    uint64_t uploads_ = 0, downloads_ = 0;
};

inline void SimState::sync() const {
    if (holder_) holder_->download(const_cast<SimState&>(*this));
}
inline void SimState::detach() {
    if (holder_) holder_->forget(this);
    holder_ = nullptr;
}
inline SimState::SimState(const SimState& o) {
    o.sync();
    copy_planes(o);
}
inline SimState::SimState(SimState&& o) noexcept {
    move_planes(o);
    token_ = o.token_, version_ = o.version_, holder_ = o.holder_;
    if (holder_) holder_->moved(&o, this);
    o.holder_ = nullptr;
    o.token_ = next_token();
}
inline SimState& SimState::operator=(const SimState& o) {
    if (this == &o) return *this;
    o.sync();
    detach();  // our device copy (if any) is overwritten
    copy_planes(o);
    ++version_;
    return *this;
}
inline SimState& SimState::operator=(SimState&& o) noexcept {
    if (this == &o) return *this;
    detach();
    move_planes(o);
    token_ = o.token_, version_ = o.version_, holder_ = o.holder_;
    if (holder_) holder_->moved(&o, this);
    o.holder_ = nullptr;
    o.token_ = next_token();
    return *this;
}
inline SimState::~SimState() { detach(); }

}  // namespace pedflow::gpu
