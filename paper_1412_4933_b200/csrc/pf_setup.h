// Host-side scenario setup (new_environment, src/state.cpp:17-75).
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <vector>

namespace pfhost {

uint64_t philox_bits(uint64_t seed, uint32_t step, uint32_t phase, uint64_t entity, uint32_t counter);
double uniform(uint64_t seed, uint32_t step, uint32_t phase, uint64_t entity, uint32_t counter);
int32_t band_height(int32_t agents_per_side, int32_t width);
// fn(begin, end) over [0, n) on up to hardware_concurrency threads (ranges of
// at least 64K).
void parallel_for(size_t n, const std::function<void(size_t, size_t)>& fn);
// fn(begin, end) over [0, n) split into `parts` ranges, run on the library's
// persistent worker threads plus the caller (no thread creation per call;
// several callers may run jobs at once). Returns when every range is done.
void pool_for(size_t n, size_t parts, const std::function<void(size_t, size_t)>& fn);
// Worker threads of the pool (hardware_concurrency - 1, at least 1).
size_t pool_threads();

// Keyed Fisher-Yates placement of one side (src/state.cpp:17-50): calls
// put(global linear cell, agent id) for the n placed agents.
void place_side(int32_t width, uint32_t group, int32_t row_begin, int32_t row_end, int32_t n, uint32_t first_id,
                uint64_t seed, const std::function<void(uint32_t cell, uint32_t id)>& put);

// The placement of one scenario: cells[0][k] / cells[1][k] = global linear
// cell of Top agent k + 1 / Bottom agent n + k + 1.
struct Placement {
    int32_t band = 0;
    std::vector<uint32_t> cells[2];
    size_t bytes() const { return (cells[0].size() + cells[1].size()) * 4; }
};

// The placement of (W, H, n, seed), computed once per process and kept in a
// small LRU cache (about 1.5 GB); concurrent requests for the same key share
// one computation. The two sides are computed in parallel.
std::shared_ptr<const Placement> placement(int32_t width, int32_t height, int32_t n, uint64_t seed);
// Start computing a placement in the background (pf_create, so that it
// overlaps the device allocation and setup); a no-op if cached or in flight.
void prefetch_placement(int32_t width, int32_t height, int32_t n, uint64_t seed);

// Both sides: Top ids 1..n in rows [0, band), Bottom ids n+1..2n in rows
// [H-band, H) (src/state.cpp:72-73). put() is called from several threads,
// once per agent.
void place_all(int32_t width, int32_t height, int32_t n, uint64_t seed,
               const std::function<void(uint32_t cell, uint32_t id, uint32_t group)>& put);

}  // namespace pfhost
