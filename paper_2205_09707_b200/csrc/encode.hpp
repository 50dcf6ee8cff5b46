// encode.hpp — GPU encode of a corpus against trained centroids + quantizer (encode.cu).
#pragma once

#include <cstdint>

#include "../../include/plaid.h"

namespace plaid {

// codes [T], residuals [T x nbits*dim/8], ivf_offsets [K + 1],
// ivf_postings [<= postings_cap]; *num_postings = ivf_offsets[K].
void encode_host(const plaid_encode_desc& in, int device, uint32_t* codes, uint8_t* residuals, uint64_t* ivf_offsets,
                 uint32_t* ivf_postings, uint64_t postings_cap, uint64_t* num_postings);

// lir::build_index (indexer.cpp:197-282) with the heavy loops on the GPU:
// centroids [k x dim], cutoffs [2^b - 1], weights [2^b], *k_out = k; the
// rest as encode_host.  Bit-identical to the reference (tests/test_gpu_build.py).
void build_index_host(const float* emb, const uint32_t* doclens, uint64_t N, uint32_t dim, uint32_t nbits, uint64_t K,
                      uint64_t iters, uint64_t seed, int device, float* centroids_out, float* cutoffs_out,
                      float* weights_out, uint64_t* k_out, uint32_t* codes, uint8_t* residuals, uint64_t* ivf_offsets,
                      uint32_t* ivf_postings, uint64_t postings_cap, uint64_t* num_postings);

}  // namespace plaid
