// The fused step kernel for grids too small to fill the GPU with the regular
// geometry (a single 480^2 scenario is 60 tiles of 16 x 256 cells): 8-row
// tiles on 64-column strips give it 480 CTAs instead of 60. The extra halo
// work is cheap next to the latency it removes (A/B, steps 5..505: C4 single
// 29.5 -> 15.8 us, C3 27.8 -> 17.9 us, C2 11.4 -> 8.6 us against 8 x 256
// tiles; 16 x 256 tiles were 44 / 40 / 14 us). See pf_bitstep.cuh / .cu.
#define PF_BITS_NS 2
#define PF_BITS_RT 8
#define PF_BITS_NAMESPACE bits_small
#include "pf_bitstep.cuh"
