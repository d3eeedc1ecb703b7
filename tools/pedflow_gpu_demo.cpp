// Drop-in demo: a run_scenario-style C++ caller (src/engine.cpp:195-231)
// driving the B200 engine through include/pedflow_gpu.hpp only.
//
//   pedflow_gpu_demo <lem|aco> <width> <height> <agents_per_side> <steps> [seed] [mode]
//
// mode:
//   batch       (default) engine.step_n(s, steps, reports): one graph-batched call
//   step        the reference's loop, `for (...) report = engine.step(state)`
//               (src/engine.cpp:216-221); the state stays on the device
//               between calls and is synced once at the end
//   interleave  step() on the state, with a second state stepped on the same
//               engine every 7th step, a copy (snapshot) taken half-way and a
//               second engine taking over for the last quarter: exercises the
//               lazy sync (the printed state must still equal the golden one)
//   phases      every step is score_phase, intention_phase, movement_phase and
//               reset_phase called one by one (PF_KERNEL_PIPELINE)
//
// stdout: moved_sum crossed_top crossed_bottom index_fnv occ_fnv (FNV-1a 64 as
// in tests/golden/make_golden.py), for comparison with the golden anchors.
// stderr: one JSON line with the timings (setup excluded from run_s, which
// covers the first upload, every step and the final download) and the
// engine's upload/download counts.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "pedflow_gpu.hpp"

static uint64_t fnv1a(const void* p, size_t n, uint64_t h = 0xcbf29ce484222325ull) {
    const auto* b = static_cast<const uint8_t*>(p);
    for (size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

static double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
    if (argc < 6) {
        std::fprintf(stderr,
                     "usage: %s <lem|aco> <width> <height> <agents_per_side> <steps> [seed] "
                     "[batch|step|interleave|phases]\n",
                     argv[0]);
        return 2;
    }
    try {
        using namespace pedflow::gpu;
        Options o;
        o.model = std::strcmp(argv[1], "lem") == 0 ? PF_MODEL_LEM : PF_MODEL_ACO;
        o.width = std::atoi(argv[2]);
        o.height = std::atoi(argv[3]);
        o.agents_per_side = std::atoi(argv[4]);
        const uint32_t steps = uint32_t(std::atoi(argv[5]));
        o.seed = argc > 6 ? std::strtoull(argv[6], nullptr, 10) : 42;
        const std::string mode = argc > 7 ? argv[7] : "batch";
        if (mode == "phases") o.kernel = PF_KERNEL_PIPELINE;
        const double t0 = now_s();
        SimState s = new_environment(o, o.seed);
        auto engine = std::make_unique<StepEngine>(o);
        const double t1 = now_s();
        std::vector<StepReport> rep(steps);
        if (mode == "phases") {
            for (uint32_t i = 0; i < steps; ++i) {  // StepEngine::step, src/engine.cpp:53-62
                engine->score_phase(s);
                engine->intention_phase(s);
                rep[i] = engine->movement_phase(s);
                engine->reset_phase(s);
            }
        } else if (mode == "step") {
            for (uint32_t i = 0; i < steps; ++i) rep[i] = engine->step(s);
        } else if (mode == "interleave") {
            SimState other = new_environment(o, o.seed + 1);
            SimState snap;
            std::unique_ptr<StepEngine> second;
            for (uint32_t i = 0; i < steps; ++i) {
                if (i == steps / 2) {
                    snap = s;  // snapshot: syncs s first
                    if (snap.step != i) throw std::logic_error("snapshot step mismatch");
                }
                if (i == 3 * steps / 4) second = std::make_unique<StepEngine>(o);
                StepEngine& e = second ? *second : *engine;
                rep[i] = e.step(s);
                if (rep[i].step != i) throw std::logic_error("report step mismatch");
                if (i % 7 == 3) engine->step(other);  // evicts s from `engine`
            }
            if (s.step != steps) throw std::logic_error("state step mismatch");
        } else if (mode == "batch") {
            engine->step_n(s, steps, rep.data());
        } else {
            std::fprintf(stderr, "unknown mode '%s'\n", mode.c_str());
            return 2;
        }
        s.sync();
        const double t2 = now_s();
        uint64_t moved = 0, top = 0, bot = 0;
        for (const auto& r : rep) {
            moved += r.moved;
            top += r.newly_crossed_top;
            bot += r.newly_crossed_bottom;
        }
        std::printf("%llu %llu %llu %016llx %016llx\n", (unsigned long long)moved, (unsigned long long)top,
                    (unsigned long long)bot, (unsigned long long)fnv1a(s.index.data(), s.index.size() * 4),
                    (unsigned long long)fnv1a(s.occupancy.data(), s.occupancy.size()));
        std::fprintf(stderr,
                     "{\"mode\": \"%s\", \"steps\": %u, \"setup_s\": %.6f, \"run_s\": %.6f, \"uploads\": %llu, "
                     "\"downloads\": %llu, \"agents\": %zu, \"cells\": %zu}\n",
                     mode.c_str(), steps, t1 - t0, t2 - t1, (unsigned long long)engine->uploads(),
                     (unsigned long long)engine->downloads(), s.agents.size(), s.index.size());
        return 0;
    } catch (const pedflow::gpu::ConfigError& e) {
        std::fprintf(stderr, "config error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
