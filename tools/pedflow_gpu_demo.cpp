// Drop-in demo: a run_scenario-style C++ caller (src/engine.cpp:195-231)
// driving the B200 engine through include/pedflow_gpu.hpp only.
//
//   pedflow_gpu_demo <lem|aco> <width> <height> <agents_per_side> <steps> [seed] [phases]
//
// With "phases" every step is StepEngine::score_phase, intention_phase,
// movement_phase and reset_phase called one by one (PF_KERNEL_PIPELINE).
//
// Prints one line: moved_sum crossed_top crossed_bottom index_fnv occ_fnv
// (FNV-1a 64 as in tests/golden/make_golden.py) so tests can compare it with
// the golden anchors.
#include <cstdio>
#include <cstdlib>
#include <cstring>
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

int main(int argc, char** argv) {
    if (argc < 6) {
        std::fprintf(stderr, "usage: %s <lem|aco> <width> <height> <agents_per_side> <steps> [seed]\n", argv[0]);
        return 2;
    }
    try {
        pedflow::gpu::Options o;
        o.model = std::strcmp(argv[1], "lem") == 0 ? PF_MODEL_LEM : PF_MODEL_ACO;
        o.width = std::atoi(argv[2]);
        o.height = std::atoi(argv[3]);
        o.agents_per_side = std::atoi(argv[4]);
        const uint32_t steps = uint32_t(std::atoi(argv[5]));
        o.seed = argc > 6 ? std::strtoull(argv[6], nullptr, 10) : 42;
        const bool phases = argc > 7 && std::strcmp(argv[7], "phases") == 0;
        if (phases) o.kernel = PF_KERNEL_PIPELINE;
        pedflow::gpu::SimState s = pedflow::gpu::new_environment(o, o.seed);
        pedflow::gpu::StepEngine engine(o);
        std::vector<pedflow::gpu::StepReport> rep(steps);
        if (phases) {
            for (uint32_t i = 0; i < steps; ++i) {  // StepEngine::step, src/engine.cpp:53-62
                engine.score_phase(s);
                engine.intention_phase(s);
                rep[i] = engine.movement_phase(s);
                engine.reset_phase(s);
            }
        } else {
            engine.step_n(s, steps, rep.data());
        }
        uint64_t moved = 0, top = 0, bot = 0;
        for (const auto& r : rep) {
            moved += r.moved;
            top += r.newly_crossed_top;
            bot += r.newly_crossed_bottom;
        }
        std::printf("%llu %llu %llu %016llx %016llx\n", (unsigned long long)moved, (unsigned long long)top,
                    (unsigned long long)bot, (unsigned long long)fnv1a(s.index.data(), s.index.size() * 4),
                    (unsigned long long)fnv1a(s.occupancy.data(), s.occupancy.size()));
        return 0;
    } catch (const pedflow::gpu::ConfigError& e) {
        std::fprintf(stderr, "config error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
