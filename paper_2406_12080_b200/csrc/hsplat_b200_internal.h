// Internal declarations shared by the host (.cpp) and device (.cu) units.
#pragma once
#include "../../include/hsplat_b200.h"

// build_bvh (build.hpp:73-149) over packed leaf Gaussians (synth.cpp's G layout).
hs_status hs_synth_build_bvh_internal(const void* leaves, uint64_t n, int nthreads, const hs_node_soa_out* out);
