// The fused step kernel for 320-column strips (10 segments); see pf_bitstep.cuh.
#define PF_BITS_NS 10
#define PF_BITS_NAMESPACE bits_ns10
#include "pf_bitstep.cuh"
