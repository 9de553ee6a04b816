// index.cu -- genome upload and GPU seed-index build.
//
// Replaces SeedIndex::build (REF src/seed_index.cpp:80-126), which rolls a
// 2s-bit key over every N-free window, std::sorts (key, pos) pairs and lays
// out a CSR of u64 keys/offsets/positions.  Here:
//   K0 planes_kernel     PackedGenome words -> bit planes (common.cuh)
//   K1a emit_kernel      one thread per window: canonical key + strand flag
//   K1b CUB radix sort   (canon<<1|flag, pos), stable -> positions ascending
//   K1c head/scan        run boundaries of equal canonical keys
//   K1d insert_kernel    one thread per distinct canonical key: position
//                        list into the pool (canon-strand windows first),
//                        open-addressing insert with atomicCAS on the key
// The index answers exactly the reference's lookup(): see common.cuh.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <string>

#include "common.cuh"
#include "device_index.h"

namespace sab {

namespace {

SA_DEV uint32_t compact_even(uint64_t x) {
    x &= 0x5555555555555555ull;
    x = (x | (x >> 1)) & 0x3333333333333333ull;
    x = (x | (x >> 2)) & 0x0F0F0F0F0F0F0F0Full;
    x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
    x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
    x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;
    return static_cast<uint32_t>(x);
}

// K0: PackedGenome layout (REF genome.hpp:50-54: base p at bits (p&31)*2 of
// word p>>5, N bit p&63 of mask word p>>6) -> planes.
__global__ void planes_kernel(const uint64_t* __restrict__ packed, uint64_t n_packed,
                              const uint64_t* __restrict__ nmask, uint64_t glen, uint4* planes,
                              uint64_t n_blocks) {
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < n_blocks;
         b += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v;
        if (b < n_packed) {
            const uint64_t w = packed[b];
            v.x = compact_even(w);
            v.y = compact_even(w >> 1);
            v.z = static_cast<uint32_t>(nmask[b >> 1] >> ((b & 1) * 32));
            const uint64_t first = b * 32;
            if (first + 32 > glen) {  // tail past the genome end reads as N
                const uint32_t valid = static_cast<uint32_t>(glen - first);
                v.z |= valid >= 32 ? 0u : ~((1u << valid) - 1u);
            }
        } else {
            v.x = v.y = 0;
            v.z = 0xffffffffu;
        }
        v.w = 0;
        planes[b] = v;
    }
}

// K1a: sort key per window (REF seed_index.cpp:96-110 rolling key; windows
// holding N are skipped, here given the sentinel so they sort last).
__global__ void emit_kernel(const uint4* __restrict__ planes, uint64_t n_windows, int s,
                            unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals,
                            unsigned long long sentinel, unsigned long long* n_valid) {
    const uint32_t smask = seed_mask32(s);
    uint32_t valid_here = 0;
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n_windows;
         p += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t lo, hi, n;
        extract32_ldg(planes, p, lo, hi, n);
        unsigned long long k;
        if (n & smask) {
            k = sentinel;
        } else {
            const uint64_t key = planar_key(lo, hi, s);
            const uint64_t rc = planar_rc_key(lo, hi, s);
            const uint64_t canon = key < rc ? key : rc;
            k = s <= 31 ? ((canon << 1) | (key != canon ? 1ull : 0ull)) : canon;
            ++valid_here;
        }
        keys[p] = k;
        vals[p] = static_cast<uint32_t>(p);
    }
    // warp-aggregated count
    for (int o = 16; o > 0; o >>= 1) valid_here += __shfl_xor_sync(0xffffffffu, valid_here, o);
    if ((threadIdx.x & 31) == 0 && valid_here) atomicAdd(n_valid, (unsigned long long)valid_here);
}

SA_DEV uint64_t canon_of(unsigned long long sk, int s) { return s <= 31 ? (sk >> 1) : sk; }

__global__ void head_kernel(const unsigned long long* __restrict__ keys, uint64_t n, int s,
                            uint32_t* __restrict__ head) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        head[i] = (i == 0 || canon_of(keys[i], s) != canon_of(keys[i - 1], s)) ? 1u : 0u;
}

__global__ void starts_kernel(const uint32_t* __restrict__ head, const uint32_t* __restrict__ rid,
                              uint64_t n, uint32_t* __restrict__ run_start) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (head[i]) run_start[rid[i]] = static_cast<uint32_t>(i);
}

// pool words a run needs: 0 for a singleton (inline), else header + list
__global__ void pool_need_kernel(const uint32_t* __restrict__ run_start, uint64_t n_runs,
                                 unsigned long long* __restrict__ need) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n_runs;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t len = run_start[r + 1] - run_start[r];
        need[r] = len > 1 ? len + 1 : 0;
    }
}

SA_DEV bool window_is_rc(const uint4* planes, uint32_t pos, int s) {
    uint32_t lo, hi, n;
    extract32_ldg(planes, pos, lo, hi, n);
    const uint64_t key = planar_key(lo, hi, s);
    const uint64_t rc = planar_rc_key(lo, hi, s);
    return rc < key;
}

// K1d
__global__ void insert_kernel(const unsigned long long* __restrict__ keys,
                              const uint32_t* __restrict__ vals,
                              const uint32_t* __restrict__ run_start, uint64_t n_runs,
                              const unsigned long long* __restrict__ pool_off,
                              const uint4* __restrict__ planes, int s, Slot* table,
                              uint64_t n_slots, uint32_t* __restrict__ pool,
                              unsigned long long* n_distinct) {
    unsigned int distinct = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n_runs;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = run_start[r], e = run_start[r + 1];
        const uint32_t len = e - b;
        const unsigned long long sk = keys[b];
        const uint64_t canon = canon_of(sk, s);
        unsigned int payload, meta;
        if (len == 1) {
            const bool flag = s <= 31 ? (sk & 1ull) : window_is_rc(planes, vals[b], s);
            payload = vals[b];
            meta = 1u | (flag ? 0x80000000u : 0u);
            distinct += 1;
        } else {
            const uint64_t off = pool_off[r];
            uint32_t n_fwd = 0;
            if (s <= 31) {  // sorted by flag within the run: canon strand first
                uint32_t lo = b, hi = e;
                while (lo < hi) {
                    uint32_t mid = lo + (hi - lo) / 2;
                    if (keys[mid] & 1ull) hi = mid;
                    else lo = mid + 1;
                }
                n_fwd = lo - b;
                for (uint32_t i = 0; i < len; ++i) pool[off + 1 + i] = vals[b + i];
            } else {  // s == 32: flag recomputed, stable partition
                uint32_t w = 0;
                for (uint32_t i = b; i < e; ++i)
                    if (!window_is_rc(planes, vals[i], s)) pool[off + 1 + w++] = vals[i];
                n_fwd = w;
                for (uint32_t i = b; i < e; ++i)
                    if (window_is_rc(planes, vals[i], s)) pool[off + 1 + w++] = vals[i];
            }
            pool[off] = n_fwd;
            // distinct forward-strand keys of this run (REF SeedIndex::distinct_seeds)
            distinct += (n_fwd > 0 ? 1u : 0u) + (n_fwd < len ? 1u : 0u);
            payload = static_cast<unsigned int>(off);
            meta = len;
        }
        uint64_t h = home_slot(canon, n_slots);
        for (;;) {
            unsigned long long old = atomicCAS(&table[h].key, kEmptyKey, (unsigned long long)canon);
            if (old == kEmptyKey) {
                table[h].payload = payload;
                table[h].meta = meta;
                break;
            }
            h = (h + 1 == n_slots) ? 0 : h + 1;
        }
    }
    for (int o = 16; o > 0; o >>= 1) distinct += __shfl_xor_sync(0xffffffffu, distinct, o);
    if ((threadIdx.x & 31) == 0 && distinct) atomicAdd(n_distinct, (unsigned long long)distinct);
}

int grid_for(uint64_t n, int threads) {
    uint64_t g = (n + threads - 1) / threads;
    if (g > 148ull * 64) g = 148ull * 64;
    if (g < 1) g = 1;
    return static_cast<int>(g);
}

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e_ = (x);                                                  \
        if (e_ != cudaSuccess) {                                               \
            err = std::string(#x) + ": " + cudaGetErrorString(e_);             \
            goto fail;                                                         \
        }                                                                      \
    } while (0)

}  // namespace

void free_device_index(DeviceIndex* ix) {
    if (ix->planes) cudaFree(ix->planes);
    if (ix->table) cudaFree(ix->table);
    if (ix->pool) cudaFree(ix->pool);
    *ix = DeviceIndex{};
}

int build_device_index(const uint64_t* h_packed, uint64_t n_packed, const uint64_t* h_nmask,
                       uint64_t n_nmask, uint64_t glen, int s, cudaStream_t st, DeviceIndex* out,
                       std::string& err) {
    DeviceIndex ix{};
    ix.glen = glen;
    ix.seed_size = s;
    ix.n_blocks = (glen + 31) / 32 + 2;
    const uint64_t n_windows = glen - s + 1;
    const unsigned long long sentinel = s <= 31 ? ((1ull << (2 * s + 1)) - 1) : ~0ull;
    const int end_bit = s <= 31 ? 2 * s + 1 : 64;

    uint64_t* d_packed = nullptr;
    uint64_t* d_nmask = nullptr;
    unsigned long long *k0 = nullptr, *k1 = nullptr, *d_count = nullptr, *pool_off = nullptr;
    uint32_t *v0 = nullptr, *v1 = nullptr, *head = nullptr, *rid = nullptr, *run_start = nullptr;
    void* temp = nullptr;
    size_t temp_bytes = 0, need = 0;
    unsigned long long n_valid = 0, pool_total = 0, last_need = 0;
    uint32_t last_head = 0, last_rid = 0;
    uint64_t n_runs = 0;
    cub::DoubleBuffer<unsigned long long> kb;
    cub::DoubleBuffer<uint32_t> vb;

    CK(cudaMalloc(&ix.planes, ix.n_blocks * sizeof(uint4)));
    CK(cudaMalloc(&d_packed, n_packed * sizeof(uint64_t) + 8));
    CK(cudaMalloc(&d_nmask, n_nmask * sizeof(uint64_t) + 8));
    CK(cudaMemcpyAsync(d_packed, h_packed, n_packed * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_nmask, h_nmask, n_nmask * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    planes_kernel<<<grid_for(ix.n_blocks, 256), 256, 0, st>>>(d_packed, n_packed, d_nmask, glen,
                                                               ix.planes, ix.n_blocks);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    cudaFree(d_packed);
    d_packed = nullptr;
    cudaFree(d_nmask);
    d_nmask = nullptr;

    CK(cudaMalloc(&k0, n_windows * sizeof(unsigned long long)));
    CK(cudaMalloc(&k1, n_windows * sizeof(unsigned long long)));
    CK(cudaMalloc(&v0, n_windows * sizeof(uint32_t)));
    CK(cudaMalloc(&v1, n_windows * sizeof(uint32_t)));
    CK(cudaMalloc(&d_count, sizeof(unsigned long long)));
    CK(cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), st));
    emit_kernel<<<grid_for(n_windows, 256), 256, 0, st>>>(ix.planes, n_windows, s, k0, v0,
                                                           sentinel, d_count);
    CK(cudaGetLastError());

    kb = cub::DoubleBuffer<unsigned long long>(k0, k1);
    vb = cub::DoubleBuffer<uint32_t>(v0, v1);
    CK(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, kb, vb, (int64_t)n_windows, 0, end_bit, st));
    CK(cudaMalloc(&temp, temp_bytes));
    CK(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, kb, vb, (int64_t)n_windows, 0, end_bit, st));
    CK(cudaMemcpyAsync(&n_valid, d_count, sizeof(n_valid), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    cudaFree(temp);
    temp = nullptr;
    ix.n_positions = n_valid;

    if (n_valid > 0) {
        // k/v of the sorted pairs live in kb.Current()/vb.Current(); reuse the
        // other buffers as scratch for the head flags and run ids.
        head = reinterpret_cast<uint32_t*>(kb.Alternate());
        rid = vb.Alternate();
        head_kernel<<<grid_for(n_valid, 256), 256, 0, st>>>(kb.Current(), n_valid, s, head);
        CK(cudaGetLastError());
        temp_bytes = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, head, rid, (int64_t)n_valid, st));
        CK(cudaMalloc(&temp, temp_bytes));
        CK(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, head, rid, (int64_t)n_valid, st));
        CK(cudaMemcpyAsync(&last_head, head + n_valid - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&last_rid, rid + n_valid - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        cudaFree(temp);
        temp = nullptr;
        n_runs = static_cast<uint64_t>(last_rid) + last_head;
        ix.n_keys = n_runs;

        CK(cudaMalloc(&run_start, (n_runs + 1) * sizeof(uint32_t)));
        starts_kernel<<<grid_for(n_valid, 256), 256, 0, st>>>(head, rid, n_valid, run_start);
        CK(cudaGetLastError());
        {
            uint32_t nv = static_cast<uint32_t>(n_valid);
            CK(cudaMemcpyAsync(run_start + n_runs, &nv, 4, cudaMemcpyHostToDevice, st));
            CK(cudaStreamSynchronize(st));
        }
        // pool offsets: exclusive sum of per-run needs (head/rid no longer used)
        CK(cudaMalloc(&pool_off, (n_runs + 1) * sizeof(unsigned long long)));
        {
            unsigned long long* needv = reinterpret_cast<unsigned long long*>(kb.Alternate());
            // Alternate holds n_windows u64 >= n_runs entries
            pool_need_kernel<<<grid_for(n_runs, 256), 256, 0, st>>>(run_start, n_runs, needv);
            CK(cudaGetLastError());
            temp_bytes = 0;
            CK(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, needv, pool_off, (int64_t)n_runs, st));
            CK(cudaMalloc(&temp, temp_bytes));
            CK(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, needv, pool_off, (int64_t)n_runs, st));
            CK(cudaMemcpyAsync(&pool_total, pool_off + n_runs - 1, 8, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(&last_need, needv + n_runs - 1, 8, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            cudaFree(temp);
            temp = nullptr;
            pool_total += last_need;
        }
        if (pool_total >= 0xffffffffull) {
            err = "position pool exceeds 2^32 entries";
            goto fail;
        }
        ix.pool_len = pool_total;
        {
            // Target fill of the open-addressing table: 35% keeps probe chains
            // at ~1.3 slots; fall back to 60% when that would take more than a
            // third of the free HBM (3.1 Gbp genomes).
            size_t free_b = 0, total_b = 0;
            cudaMemGetInfo(&free_b, &total_b);
            const uint64_t sparse = n_runs * 100 / 35 + 64;
            ix.n_slots = sparse * sizeof(Slot) <= free_b / 3 ? sparse : n_runs * 100 / 60 + 64;
        }
        CK(cudaMalloc(&ix.table, ix.n_slots * sizeof(Slot)));
        CK(cudaMemsetAsync(ix.table, 0xff, ix.n_slots * sizeof(Slot), st));
        CK(cudaMalloc(&ix.pool, (pool_total + 1) * sizeof(uint32_t)));
        CK(cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), st));
        insert_kernel<<<grid_for(n_runs, 128), 128, 0, st>>>(kb.Current(), vb.Current(), run_start,
                                                              n_runs, pool_off, ix.planes, s,
                                                              ix.table, ix.n_slots, ix.pool,
                                                              d_count);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&ix.n_distinct, d_count, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    } else {
        ix.n_slots = 64;
        CK(cudaMalloc(&ix.table, ix.n_slots * sizeof(Slot)));
        CK(cudaMemsetAsync(ix.table, 0xff, ix.n_slots * sizeof(Slot), st));
        CK(cudaMalloc(&ix.pool, sizeof(uint32_t)));
        CK(cudaStreamSynchronize(st));
    }
    cudaFree(k0);
    cudaFree(k1);
    cudaFree(v0);
    cudaFree(v1);
    cudaFree(d_count);
    if (run_start) cudaFree(run_start);
    if (pool_off) cudaFree(pool_off);
    ix.device_bytes = ix.n_blocks * sizeof(uint4) + ix.n_slots * sizeof(Slot) +
                      (ix.pool_len + 1) * sizeof(uint32_t);
    *out = ix;
    (void)need;
    return 0;

fail:
    if (d_packed) cudaFree(d_packed);
    if (d_nmask) cudaFree(d_nmask);
    if (k0) cudaFree(k0);
    if (k1) cudaFree(k1);
    if (v0) cudaFree(v0);
    if (v1) cudaFree(v1);
    if (d_count) cudaFree(d_count);
    if (run_start) cudaFree(run_start);
    if (pool_off) cudaFree(pool_off);
    if (temp) cudaFree(temp);
    free_device_index(&ix);
    return 2;
}

}  // namespace sab
