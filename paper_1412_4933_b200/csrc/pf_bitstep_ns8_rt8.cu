// The fused step kernel with 8-row tiles on 256-column strips, for grids too
// small to fill the GPU with 16-row tiles (single 480^2 scenarios); see
// pf_bitstep.cuh and pf_bitstep.cu.
#define PF_BITS_NS 8
#define PF_BITS_RT 8
#define PF_BITS_NAMESPACE bits_ns8_rt8
#include "pf_bitstep.cuh"
