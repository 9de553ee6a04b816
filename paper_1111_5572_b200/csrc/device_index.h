// device_index.h -- the per-GPU replica: genome bit planes + seed hash table
// + position pool (layouts in common.cuh).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace sab {

struct Slot;

struct DeviceIndex {
    uint4* planes = nullptr;  // n_blocks = ceil(glen/32) + 2
    uint64_t n_blocks = 0;
    uint64_t glen = 0;
    int seed_size = 0;
    Slot* table = nullptr;
    uint64_t n_slots = 0;
    uint32_t* pool = nullptr;
    uint64_t pool_len = 0;
    uint64_t n_keys = 0;       // distinct canonical keys (table entries)
    unsigned long long n_distinct = 0;  // distinct forward keys (REF distinct_seeds)
    uint64_t n_positions = 0;  // N-free windows (REF SeedIndex::total_positions)
    uint64_t device_bytes = 0;
};

int build_device_index(const uint64_t* h_packed, uint64_t n_packed, const uint64_t* h_nmask,
                       uint64_t n_nmask, uint64_t glen, int s, cudaStream_t st, DeviceIndex* out,
                       std::string& err);
void free_device_index(DeviceIndex* ix);

}  // namespace sab
