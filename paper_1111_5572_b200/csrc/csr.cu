// csr.cu -- the reference's CSR seed index, built on the GPU.
//
// REF src/seed_index.cpp:80-126 (SeedIndex::build) rolls a 2s-bit packed key
// (first base in the high bits, REF :51-60) over every N-free window,
// std::sorts (key, position) pairs and keeps three u64 arrays: sorted distinct
// keys, offsets (keys + 1) and positions ascending per key
// (include/seedaln/seed_index.hpp:66-71).  Those arrays are what an SNAPIDX1
// index file stores (REF :145-170), so this is the path behind writing and
// verifying reference-format index files; the aligner itself uses the hash
// table of index.cu.
//
//   C0 hist_kernel      window counts per key bin (top <= 16 key bits)
//   host                contiguous bin ranges -> partitions within budget
//   per partition:
//     C1 count/write    ordered compaction of the partition's windows:
//                       (packed key, position), positions ascending
//     C2 CUB radix sort stable over the 2s key bits -> ascending per key
//     C3 CUB run-length encode -> distinct keys + run lengths
//     D2H               appended to the host CSR (partitions are key ranges,
//                       so concatenation is globally sorted)
#include <cuda_runtime.h>

#include <algorithm>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>
#include <string>
#include <vector>

#include "common.cuh"
#include "device_index.h"

namespace sab {

namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = 16;  // consecutive windows per thread
constexpr uint64_t kPerBlock = static_cast<uint64_t>(kThreads) * kPerThread;

// Packed key of window p (REF seed_index.cpp:96-110), false when it holds N.
SA_DEV bool window_packed(const uint4* planes, uint64_t p, int s, uint64_t& key) {
    uint32_t lo, hi, n;
    extract32_ldg(planes, p, lo, hi, n);
    if (n & seed_mask32(s)) return false;
    key = packed_key(lo, hi, s);
    return true;
}

__global__ void __launch_bounds__(kThreads) hist_kernel(const uint4* __restrict__ planes, uint64_t n_windows,
                                                        int s, int bin_shift, unsigned long long* bins) {
    for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < n_windows;
         p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t k;
        if (window_packed(planes, p, s, k)) atomicAdd(bins + (k >> bin_shift), 1ull);
    }
}

SA_DEV bool in_part(uint64_t k, int bin_shift, uint64_t bin_lo, uint64_t bin_hi) {
    const uint64_t b = k >> bin_shift;
    return b >= bin_lo && b < bin_hi;
}

__global__ void __launch_bounds__(kThreads) count_kernel(const uint4* __restrict__ planes, uint64_t n_windows,
                                                         int s, int bin_shift, uint64_t bin_lo, uint64_t bin_hi,
                                                         unsigned long long* block_counts) {
    typedef cub::BlockReduce<unsigned int, kThreads> Reduce;
    __shared__ typename Reduce::TempStorage tmp;
    const uint64_t base = blockIdx.x * kPerBlock + static_cast<uint64_t>(threadIdx.x) * kPerThread;
    unsigned int c = 0;
    for (int j = 0; j < kPerThread; ++j) {
        uint64_t k;
        const uint64_t p = base + j;
        if (p < n_windows && window_packed(planes, p, s, k) && in_part(k, bin_shift, bin_lo, bin_hi)) ++c;
    }
    const unsigned int tot = Reduce(tmp).Sum(c);
    if (threadIdx.x == 0) block_counts[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kThreads) write_kernel(const uint4* __restrict__ planes, uint64_t n_windows,
                                                         int s, int bin_shift, uint64_t bin_lo, uint64_t bin_hi,
                                                         const unsigned long long* block_offs,
                                                         unsigned long long* __restrict__ keys,
                                                         uint32_t* __restrict__ pos) {
    typedef cub::BlockScan<unsigned int, kThreads> Scan;
    __shared__ typename Scan::TempStorage tmp;
    const uint64_t base = blockIdx.x * kPerBlock + static_cast<uint64_t>(threadIdx.x) * kPerThread;
    uint64_t kk[kPerThread];
    unsigned int c = 0, m = 0;
    for (int j = 0; j < kPerThread; ++j) {
        uint64_t k;
        const uint64_t p = base + j;
        if (p < n_windows && window_packed(planes, p, s, k) && in_part(k, bin_shift, bin_lo, bin_hi)) {
            m |= 1u << j;
            kk[c++] = k;
        }
    }
    unsigned int pre;
    Scan(tmp).ExclusiveSum(c, pre);
    uint64_t o = block_offs[blockIdx.x] + pre;
    unsigned int q = 0;
    for (int j = 0; j < kPerThread; ++j) {
        if (m & (1u << j)) {
            keys[o] = kk[q++];
            pos[o] = static_cast<uint32_t>(base + j);
            ++o;
        }
    }
}

struct Bufs {  // temporaries, freed on scope exit
    std::vector<void*> p;
    template <typename T>
    cudaError_t alloc(T** out, uint64_t count) {
        void* q = nullptr;
        cudaError_t e = cudaMalloc(&q, std::max<uint64_t>(count, 1) * sizeof(T));
        if (e == cudaSuccess) {
            p.push_back(q);
            *out = static_cast<T*>(q);
        }
        return e;
    }
    ~Bufs() {
        for (void* q : p) cudaFree(q);
    }
};

}  // namespace

#define CSR_TRY(x)                                                             \
    do {                                                                       \
        cudaError_t e_ = (x);                                                  \
        if (e_ != cudaSuccess) {                                               \
            err = std::string(#x) + ": " + cudaGetErrorString(e_);             \
            return 2;                                                          \
        }                                                                      \
    } while (0)

int build_csr_index(const uint4* d_planes, uint64_t glen, int s, cudaStream_t st, CsrIndex* out,
                    std::string& err) {
    out->keys.clear();
    out->offsets.assign(1, 0);
    out->positions.clear();
    if (s < 1 || s > 32 || glen < static_cast<uint64_t>(s)) {
        err = "bad seed size for the genome";
        return 1;
    }
    const uint64_t n_windows = glen - s + 1;
    const int key_bits = 2 * s;
    const int bin_bits = std::min(16, key_bits);
    const int bin_shift = key_bits - bin_bits;
    const uint64_t n_bins = 1ull << bin_bits;
    Bufs b;
    unsigned long long* bins = nullptr;
    CSR_TRY(b.alloc(&bins, n_bins));
    CSR_TRY(cudaMemsetAsync(bins, 0, n_bins * sizeof(unsigned long long), st));
    {
        const uint64_t g = std::min<uint64_t>((n_windows + kThreads - 1) / kThreads, 148ull * 64);
        hist_kernel<<<static_cast<int>(std::max<uint64_t>(g, 1)), kThreads, 0, st>>>(d_planes, n_windows, s,
                                                                                     bin_shift, bins);
        CSR_TRY(cudaGetLastError());
    }
    std::vector<unsigned long long> h_bins(n_bins);
    CSR_TRY(cudaMemcpyAsync(h_bins.data(), bins, n_bins * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CSR_TRY(cudaStreamSynchronize(st));
    uint64_t total = 0;
    for (auto v : h_bins) total += v;
    if (total == 0) return 0;

    // partitions: contiguous bin ranges of at most `cap` windows (~36 B each)
    size_t free_b = 0, total_b = 0;
    CSR_TRY(cudaMemGetInfo(&free_b, &total_b));
    uint64_t cap = std::max<uint64_t>(free_b / 2 / 40, 1 << 20);
    uint64_t biggest = *std::max_element(h_bins.begin(), h_bins.end());
    cap = std::max(cap, static_cast<uint64_t>(biggest));
    cap = std::min(cap, total);
    std::vector<uint64_t> cuts{0};
    uint64_t acc = 0;
    for (uint64_t i = 0; i < n_bins; ++i) {
        if (acc + h_bins[i] > cap && acc > 0) {
            cuts.push_back(i);
            acc = 0;
        }
        acc += h_bins[i];
    }
    cuts.push_back(n_bins);

    const uint64_t n_eblocks = (n_windows + kPerBlock - 1) / kPerBlock;
    unsigned long long *bcount = nullptr, *boff = nullptr, *k0 = nullptr, *k1 = nullptr, *ukeys = nullptr;
    uint32_t *v0 = nullptr, *v1 = nullptr, *runs = nullptr, *nruns = nullptr;
    CSR_TRY(b.alloc(&bcount, n_eblocks + 1));
    CSR_TRY(b.alloc(&boff, n_eblocks + 1));
    CSR_TRY(b.alloc(&k0, cap));
    CSR_TRY(b.alloc(&k1, cap));
    CSR_TRY(b.alloc(&v0, cap));
    CSR_TRY(b.alloc(&v1, cap));
    CSR_TRY(b.alloc(&ukeys, cap));
    CSR_TRY(b.alloc(&runs, cap));
    CSR_TRY(b.alloc(&nruns, 1));
    size_t temp_bytes = 0;
    void* temp = nullptr;
    {
        size_t a = 0, c = 0, d = 0;
        cub::DoubleBuffer<unsigned long long> kb(k0, k1);
        cub::DoubleBuffer<uint32_t> vb(v0, v1);
        CSR_TRY(cub::DeviceRadixSort::SortPairs(nullptr, a, kb, vb, static_cast<int64_t>(cap), 0, key_bits, st));
        CSR_TRY(cub::DeviceScan::ExclusiveSum(nullptr, c, bcount, boff, static_cast<int64_t>(n_eblocks + 1), st));
        CSR_TRY(cub::DeviceRunLengthEncode::Encode(nullptr, d, k0, ukeys, runs, nruns, static_cast<int64_t>(cap), st));
        temp_bytes = std::max(a, std::max(c, d));
        unsigned char* t = nullptr;
        CSR_TRY(b.alloc(&t, temp_bytes));
        temp = t;
    }
    out->keys.reserve(out->keys.size());
    out->positions.resize(total);
    uint64_t pos_at = 0;
    std::vector<unsigned long long> h_keys;
    std::vector<uint32_t> h_runs, h_pos;
    for (size_t part = 0; part + 1 < cuts.size(); ++part) {
        const uint64_t lo = cuts[part], hi = cuts[part + 1];
        uint64_t n_p = 0;
        for (uint64_t i = lo; i < hi; ++i) n_p += h_bins[i];
        if (n_p == 0) continue;
        count_kernel<<<static_cast<int>(n_eblocks), kThreads, 0, st>>>(d_planes, n_windows, s, bin_shift, lo, hi,
                                                                      bcount);
        CSR_TRY(cudaGetLastError());
        CSR_TRY(cudaMemsetAsync(bcount + n_eblocks, 0, sizeof(unsigned long long), st));
        CSR_TRY(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, bcount, boff, static_cast<int64_t>(n_eblocks + 1), st));
        write_kernel<<<static_cast<int>(n_eblocks), kThreads, 0, st>>>(d_planes, n_windows, s, bin_shift, lo, hi,
                                                                      boff, k0, v0);
        CSR_TRY(cudaGetLastError());
        cub::DoubleBuffer<unsigned long long> kb(k0, k1);
        cub::DoubleBuffer<uint32_t> vb(v0, v1);
        CSR_TRY(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, kb, vb, static_cast<int64_t>(n_p), 0, key_bits, st));
        CSR_TRY(cub::DeviceRunLengthEncode::Encode(temp, temp_bytes, kb.Current(), ukeys, runs, nruns,
                                                   static_cast<int64_t>(n_p), st));
        uint32_t h_nruns = 0;
        CSR_TRY(cudaMemcpyAsync(&h_nruns, nruns, sizeof(h_nruns), cudaMemcpyDeviceToHost, st));
        CSR_TRY(cudaStreamSynchronize(st));
        h_keys.resize(h_nruns);
        h_runs.resize(h_nruns);
        h_pos.resize(n_p);
        CSR_TRY(cudaMemcpyAsync(h_keys.data(), ukeys, h_nruns * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CSR_TRY(cudaMemcpyAsync(h_runs.data(), runs, h_nruns * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        CSR_TRY(cudaMemcpyAsync(h_pos.data(), vb.Current(), n_p * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        CSR_TRY(cudaStreamSynchronize(st));
        for (uint32_t i = 0; i < h_nruns; ++i) {
            out->keys.push_back(h_keys[i]);
            out->offsets.push_back(out->offsets.back() + h_runs[i]);
        }
        for (uint64_t i = 0; i < n_p; ++i) out->positions[pos_at + i] = h_pos[i];
        pos_at += n_p;
    }
    return 0;
}

}  // namespace sab
