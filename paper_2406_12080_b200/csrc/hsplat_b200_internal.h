// Internal declarations shared by the host (.cpp) and device (.cu) units.
#pragma once
#include "../../include/hsplat_b200.h"

// build_bvh (build.hpp:73-149) over packed leaf Gaussians (synth.cpp's G layout).
hs_status hs_synth_build_bvh_internal(const void* leaves, uint64_t n, int nthreads, const hs_node_soa_out* out);

// consolidate's global root over k forest roots (scene.hpp:264-279, 307-313);
// records are 59 floats {mean3, scale3, quat wxyz 4, falloff, sh48}.
void hs_merge_root_internal(const float* gin, uint32_t k, const float* bmin, const float* bmax, float* root,
                            float* root_bmin, float* root_bmax, float* gout);
