// Host-side scenario setup (new_environment, src/state.cpp:17-75).
#pragma once

#include <cstdint>
#include <functional>

namespace pfhost {

uint64_t philox_bits(uint64_t seed, uint32_t step, uint32_t phase, uint64_t entity, uint32_t counter);
double uniform(uint64_t seed, uint32_t step, uint32_t phase, uint64_t entity, uint32_t counter);
int32_t band_height(int32_t agents_per_side, int32_t width);

// Keyed Fisher-Yates placement of one side (src/state.cpp:17-50): calls
// put(global linear cell, agent id) for the n placed agents.
void place_side(int32_t width, uint32_t group, int32_t row_begin, int32_t row_end, int32_t n, uint32_t first_id,
                uint64_t seed, const std::function<void(uint32_t cell, uint32_t id)>& put);

// Both sides: Top ids 1..n in rows [0, band), Bottom ids n+1..2n in rows
// [H-band, H) (src/state.cpp:72-73).
void place_all(int32_t width, int32_t height, int32_t n, uint64_t seed,
               const std::function<void(uint32_t cell, uint32_t id, uint32_t group)>& put);

}  // namespace pfhost
