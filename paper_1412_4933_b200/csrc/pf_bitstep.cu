// Strip-width dispatch of the fused step kernel (pf_bitstep.cuh).
//
// A work unit of S1/S2 is one 32-cell segment-row of a tile plus the halo
// segments on each side of its strip, and a CTA runs one unit per thread.
// 10-segment strips (320 columns) keep 240 of the 256 threads busy in S1
// (8-segment strips: 200) and pay 2 halo segments per 10 instead of per 8,
// but waste whole segments when the grid width is not a multiple of 320:
// for LEM the strip width with fewer units per row wins (A/B at step 150: C5
// LEM -9% with 10; 480-wide grids: 8, since 10 would pad 15 segments to 20).
// ACO, bound by its pheromone stream, keeps 8 (C5 ACO +0.4% with 10, and
// +22% with 10 since the 32-row tiles came); with fp32 pheromone storage it
// takes the LEM rule (C5: 10, -2%: twice the bytes in flight per lane).
#include "pf_internal.h"

namespace pfk {
namespace bits_ns8 {
int configure();
int launch(const StepArgs& a, int slot, int parity, cudaStream_t s);
}  // namespace bits_ns8
namespace bits_ns10 {
int configure();
int launch(const StepArgs& a, int slot, int parity, cudaStream_t s);
}  // namespace bits_ns10
namespace bits_small {
int configure();
int launch(const StepArgs& a, int slot, int parity, cudaStream_t s);
}  // namespace bits_small

int bits_strip_segments(int width, int model, bool tau_f32) {
    if (model == 1 && !tau_f32) return 8;
    const int ws = (width + 31) / 32;
    auto units = [ws](int ns) { return ((ws + ns - 1) / ns) * (ns + 2); };
    return units(10) < units(8) ? 10 : 8;
}

int configure_step_bits() { return bits_ns8::configure() | bits_ns10::configure() | bits_small::configure(); }

// Grids with fewer than 2 x SMs 16-row tiles (a single 480^2 scenario: 60
// tiles) run about one tile per CTA on a fraction of the GPU, so their step
// time is one tile's latency: they take 8-row tiles on 64-column strips (8x
// the CTAs, pf_bitstep_small.cu). Sweep (tools/small_tiles_sweep.py, 480^2
// x R, 102,400 agents): x1 46 -> 17 us, x2 46 -> 28, x4 51 -> 37; x8 is
// even (2-agent-dense LEM and sparse grids lose there). The occupancy-plane
// pitch (strips of 8 or 10 segments) also fits the 2-segment strips.
int launch_step_bits(const StepArgs& a, int slot, int parity, cudaStream_t s) {
    if (a.cluster > 0 && !a.peer[0].cell && !a.peer[1].cell) {
        if (const int n = launch_cluster_lem(a, slot, parity, s)) return n;
    }
    const long long strips = (a.k.W + 255) / 256, tiles16 = strips * ((a.rows_owned + 15) / 16) * a.replicas;
    if (a.small_tiles == 1 || (a.small_tiles < 0 && tiles16 < 2LL * a.num_sms)) return bits_small::launch(a, slot, parity, s);
    if (a.strip_segs == 10) return bits_ns10::launch(a, slot, parity, s);
    return bits_ns8::launch(a, slot, parity, s);
}

}  // namespace pfk
