// The fused step kernel for 256-column strips (8 segments); see pf_bitstep.cuh.
#define PF_BITS_NS 8
#define PF_BITS_NAMESPACE bits_ns8
#include "pf_bitstep.cuh"
