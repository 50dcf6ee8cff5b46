// encode.hpp — GPU encode of a corpus against trained centroids + quantizer (encode.cu).
#pragma once

#include <cstdint>

#include "../../include/plaid.h"

namespace plaid {

// codes [T], residuals [T x nbits*dim/8], ivf_offsets [K + 1],
// ivf_postings [<= postings_cap]; *num_postings = ivf_offsets[K].
void encode_host(const plaid_encode_desc& in, int device, uint32_t* codes, uint8_t* residuals, uint64_t* ivf_offsets,
                 uint32_t* ivf_postings, uint64_t postings_cap, uint64_t* num_postings);

}  // namespace plaid
