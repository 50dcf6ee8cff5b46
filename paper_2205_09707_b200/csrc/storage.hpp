// storage.hpp — on-disk index format (storage.cu, FORMAT.md).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/plaid.h"

namespace plaid {

class DeviceIndex;

constexpr int kFormatVersion = 1;

// File digest of FORMAT.md (64 KiB blocks, 32 word lanes per block, FNV-1a 64).
uint64_t checksum_host(const void* data, uint64_t bytes);
uint64_t checksum_device(const void* d_data, uint64_t bytes, cudaStream_t st);

// manifest.json + the six little-endian arrays; partial files are removed on failure.
void save_index(const plaid_index_desc& d, const std::string& dir, uint64_t rng_seed);
// mmap -> HBM upload -> checksums of the uploaded arrays on the GPU
// (-> validate_index when PLAID_OPEN_VALIDATE).  Caller owns the result.
DeviceIndex* open_index(const std::string& dir, int device, uint32_t flags);

}  // namespace plaid
