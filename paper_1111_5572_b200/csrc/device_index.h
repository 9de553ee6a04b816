// device_index.h -- the per-GPU replica: genome bit planes + seed hash table
// + position pool (layouts in common.cuh).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

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

// PackedGenome words -> device bit planes (ceil(glen/32) + 2 uint4 blocks,
// all-N padding), synchronous on st.  0 ok, 2 CUDA error (message in err).
int upload_planes(const uint64_t* h_packed, uint64_t n_packed, const uint64_t* h_nmask, uint64_t n_nmask,
                  uint64_t glen, cudaStream_t st, uint4** d_planes, std::string& err);

// The reference's CSR seed index (REF src/seed_index.cpp:80-126,
// include/seedaln/seed_index.hpp:66-71) computed on the GPU from device
// planes: keys = sorted distinct packed forward keys, offsets (keys+1),
// positions ascending per key -- every N-free window.  Built in key-range
// partitions sized to free HBM and streamed to the host vectors.
struct CsrIndex {
    std::vector<uint64_t> keys, offsets, positions;
};
int build_csr_index(const uint4* d_planes, uint64_t glen, int s, cudaStream_t st, CsrIndex* out,
                    std::string& err);

}  // namespace sab
