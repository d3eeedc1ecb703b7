// The fused step kernel for 320-column strips (10 segments) and 32-row tiles:
// the LEM geometry for wide grids (A/B at step 150, C5 LEM: -9% for 10 segments
// over 8, then -4% for 32 rows over 16). See pf_bitstep.cuh / pf_bitstep.cu.
#define PF_BITS_NS 10
#define PF_BITS_RT 32
#define PF_BITS_NAMESPACE bits_ns10
#include "pf_bitstep.cuh"
