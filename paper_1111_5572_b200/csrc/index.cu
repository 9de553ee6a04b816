// index.cu -- genome upload and GPU seed-index build.
//
// Replaces SeedIndex::build (REF src/seed_index.cpp:80-126), which rolls a
// 2s-bit key over every N-free window, std::sorts (key, pos) pairs and lays
// out a CSR of u64 keys/offsets/positions.  Here:
//   K0 planes_kernel      PackedGenome words -> bit planes (common.cuh)
//   per key-hash partition p of P (P = 1 up to a few hundred Mbp; more for
//   3.1 Gbp genomes, so build temporaries stay bounded):
//     K1a count/write     ordered compaction of the N-free windows whose
//                         canonical key falls in p: (canon<<1|strand, pos),
//                         positions ascending (block scan, deterministic)
//     K1b CUB radix sort  stable -> positions stay ascending per key
//     K1c head/scan       run boundaries of equal canonical keys
//     K1d insert_kernel   one thread per distinct key: position list into the
//                         pool (canon-strand windows first), open-addressing
//                         insert with atomicCAS on the key
// The table is sized from the window count (an upper bound on distinct keys)
// before the first partition; the pool grows between partitions if needed.
// The index answers exactly the reference's lookup(): see common.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <string>

#include "common.cuh"
#include "device_index.h"

namespace sab {

namespace {

constexpr int kEmitThreads = 256;
constexpr int kEmitPerThread = 16;  // consecutive windows per thread
constexpr uint64_t kEmitPerBlock = static_cast<uint64_t>(kEmitThreads) * kEmitPerThread;

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

// Window p's sort key, or false when the window holds N (REF
// seed_index.cpp:96-110 skips those) or its key is outside partition `part`.
SA_DEV bool window_key(const uint4* planes, uint64_t p, int s, uint32_t part, uint32_t n_parts,
                       unsigned long long& sk) {
    uint32_t lo, hi, n;
    extract32_ldg(planes, p, lo, hi, n);
    if (n & seed_mask32(s)) return false;
    const uint64_t key = planar_key(lo, hi, s);
    const uint64_t rc = planar_rc_key(lo, hi, s);
    const uint64_t canon = key < rc ? key : rc;
    if (n_parts > 1 && static_cast<uint32_t>(((mix64(canon) >> 32) * n_parts) >> 32) != part) return false;
    sk = s <= 31 ? ((canon << 1) | (key != canon ? 1ull : 0ull)) : canon;
    return true;
}

// K1a (count): windows of partition `part` per block of kEmitPerBlock windows.
__global__ void __launch_bounds__(kEmitThreads) count_part_kernel(const uint4* __restrict__ planes,
                                                                  uint64_t n_windows, int s, uint32_t part,
                                                                  uint32_t n_parts,
                                                                  unsigned long long* block_counts) {
    typedef cub::BlockReduce<unsigned int, kEmitThreads> Reduce;
    __shared__ typename Reduce::TempStorage tmp;
    const uint64_t base = blockIdx.x * kEmitPerBlock + static_cast<uint64_t>(threadIdx.x) * kEmitPerThread;
    unsigned int c = 0;
    for (int j = 0; j < kEmitPerThread; ++j) {
        const uint64_t p = base + j;
        unsigned long long sk;
        if (p < n_windows && window_key(planes, p, s, part, n_parts, sk)) ++c;
    }
    const unsigned int tot = Reduce(tmp).Sum(c);
    if (threadIdx.x == 0) block_counts[blockIdx.x] = tot;
}

// K1a (write): same walk; each thread writes its matches at its block offset
// plus its exclusive prefix, so output keeps genome position order.
__global__ void __launch_bounds__(kEmitThreads) write_part_kernel(const uint4* __restrict__ planes,
                                                                  uint64_t n_windows, int s, uint32_t part,
                                                                  uint32_t n_parts,
                                                                  const unsigned long long* block_offs,
                                                                  unsigned long long* __restrict__ keys,
                                                                  uint32_t* __restrict__ vals) {
    typedef cub::BlockScan<unsigned int, kEmitThreads> Scan;
    __shared__ typename Scan::TempStorage tmp;
    const uint64_t base = blockIdx.x * kEmitPerBlock + static_cast<uint64_t>(threadIdx.x) * kEmitPerThread;
    unsigned long long sk[kEmitPerThread];
    unsigned int c = 0, m = 0;
    for (int j = 0; j < kEmitPerThread; ++j) {
        const uint64_t p = base + j;
        if (p < n_windows && window_key(planes, p, s, part, n_parts, sk[c])) {
            m |= 1u << j;
            ++c;
        }
    }
    unsigned int pre;
    Scan(tmp).ExclusiveSum(c, pre);
    uint64_t o = block_offs[blockIdx.x] + pre;
    unsigned int k = 0;
    for (int j = 0; j < kEmitPerThread; ++j) {
        if (m & (1u << j)) {
            keys[o] = sk[k++];
            vals[o] = static_cast<uint32_t>(base + j);
            ++o;
        }
    }
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
                              const unsigned long long* __restrict__ pool_off, uint64_t pool_base,
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
            const uint64_t off = pool_base + pool_off[r];
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

struct Scratch {  // build temporaries, freed at the end
    void* p[12] = {};
    int n = 0;
    template <typename T>
    cudaError_t alloc(T** out, uint64_t count) {
        void* q = nullptr;
        cudaError_t e = cudaMalloc(&q, std::max<uint64_t>(count, 1) * sizeof(T));
        if (e == cudaSuccess) {
            p[n++] = q;
            *out = static_cast<T*>(q);
        }
        return e;
    }
    ~Scratch() {
        for (int i = 0; i < n; ++i) cudaFree(p[i]);
    }
};

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e_ = (x);                                                  \
        if (e_ != cudaSuccess) {                                               \
            err = std::string(#x) + ": " + cudaGetErrorString(e_);             \
            free_device_index(&ix);                                            \
            return 2;                                                          \
        }                                                                      \
    } while (0)

}  // namespace

void free_device_index(DeviceIndex* ix) {
    if (ix->planes) cudaFree(ix->planes);
    if (ix->table) cudaFree(ix->table);
    if (ix->pool) cudaFree(ix->pool);
    *ix = DeviceIndex{};
}

int upload_planes(const uint64_t* h_packed, uint64_t n_packed, const uint64_t* h_nmask, uint64_t n_nmask,
                  uint64_t glen, cudaStream_t st, uint4** d_planes, std::string& err) {
    const uint64_t n_blocks = (glen + 31) / 32 + 2;
    *d_planes = nullptr;
#define UP(x)                                                              \
    do {                                                                   \
        cudaError_t e_ = (x);                                              \
        if (e_ != cudaSuccess) {                                           \
            err = std::string(#x) + ": " + cudaGetErrorString(e_);         \
            if (*d_planes) cudaFree(*d_planes);                            \
            *d_planes = nullptr;                                           \
            return 2;                                                      \
        }                                                                  \
    } while (0)
    UP(cudaMalloc(d_planes, n_blocks * sizeof(uint4)));
    Scratch up;
    uint64_t *d_packed = nullptr, *d_nmask = nullptr;
    UP(up.alloc(&d_packed, n_packed + 1));
    UP(up.alloc(&d_nmask, n_nmask + 1));
    UP(cudaMemcpyAsync(d_packed, h_packed, n_packed * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    UP(cudaMemcpyAsync(d_nmask, h_nmask, n_nmask * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    planes_kernel<<<grid_for(n_blocks, 256), 256, 0, st>>>(d_packed, n_packed, d_nmask, glen, *d_planes, n_blocks);
    UP(cudaGetLastError());
    UP(cudaStreamSynchronize(st));
#undef UP
    return 0;
}

int build_device_index(const uint64_t* h_packed, uint64_t n_packed, const uint64_t* h_nmask,
                       uint64_t n_nmask, uint64_t glen, int s, cudaStream_t st, DeviceIndex* out,
                       std::string& err) {
    DeviceIndex ix{};
    ix.glen = glen;
    ix.seed_size = s;
    ix.n_blocks = (glen + 31) / 32 + 2;
    const uint64_t n_windows = glen - s + 1;
    const int end_bit = s <= 31 ? 2 * s + 1 : 64;

    // ---- genome planes
    if (upload_planes(h_packed, n_packed, h_nmask, n_nmask, glen, st, &ix.planes, err) != 0) {
        free_device_index(&ix);
        return 2;
    }

    // ---- table sized from the window count (upper bound on distinct keys):
    // 35% target load keeps probe chains ~1.3 slots; 60% when that would take
    // more than a third of the free HBM (3.1 Gbp genomes)
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    {
        const uint64_t sparse = n_windows * 100 / 35 + 64;
        ix.n_slots = sparse * sizeof(Slot) <= free_b / 3 ? sparse : n_windows * 100 / 60 + 64;
    }
    CK(cudaMalloc(&ix.table, ix.n_slots * sizeof(Slot)));
    CK(cudaMemsetAsync(ix.table, 0xff, ix.n_slots * sizeof(Slot), st));

    // ---- partitions: ~40 B of temporaries per window of a partition
    CK(cudaMemGetInfo(&free_b, &total_b));
    const uint64_t budget = free_b / 2;
    uint32_t n_parts = static_cast<uint32_t>((n_windows * 48 + budget - 1) / budget);
    if (n_parts < 1) n_parts = 1;
    if (const char* e = getenv("SA_INDEX_PARTS")) {  // test hook: force a partitioned build
        const long f = strtol(e, nullptr, 10);
        if (f > static_cast<long>(n_parts) && f < 65536) n_parts = static_cast<uint32_t>(f);
    }
    const uint64_t cap = n_windows / n_parts + n_windows / (8 * n_parts) + 4096;  // hash imbalance slack
    uint64_t pool_cap = std::max<uint64_t>(1 << 20, n_windows / 8);
    CK(cudaMalloc(&ix.pool, pool_cap * sizeof(uint32_t)));
    uint64_t pool_used = 0;

    Scratch tmp;
    const uint64_t n_eblocks = (n_windows + kEmitPerBlock - 1) / kEmitPerBlock;
    unsigned long long *bcount = nullptr, *boff = nullptr, *k0 = nullptr, *k1 = nullptr, *pool_off = nullptr,
                       *d_count = nullptr;
    uint32_t *v0 = nullptr, *v1 = nullptr, *run_start = nullptr;
    CK(tmp.alloc(&bcount, n_eblocks + 1));
    CK(tmp.alloc(&boff, n_eblocks + 1));
    CK(tmp.alloc(&k0, cap + 1));  // +1: the run-need vector (aliased on k0/k1) has n_runs+1 entries
    CK(tmp.alloc(&k1, cap + 1));
    CK(tmp.alloc(&v0, cap));
    CK(tmp.alloc(&v1, cap));
    CK(tmp.alloc(&run_start, cap + 1));
    CK(tmp.alloc(&pool_off, cap + 1));
    CK(tmp.alloc(&d_count, 2));
    CK(cudaMemsetAsync(d_count, 0, 2 * sizeof(unsigned long long), st));
    void* temp = nullptr;
    size_t temp_bytes = 0;
    {
        size_t a = 0, b = 0, c = 0;
        cub::DoubleBuffer<unsigned long long> kb(k0, k1);
        cub::DoubleBuffer<uint32_t> vb(v0, v1);
        CK(cub::DeviceRadixSort::SortPairs(nullptr, a, kb, vb, (int64_t)cap, 0, end_bit, st));
        CK(cub::DeviceScan::ExclusiveSum(nullptr, b, v0, v1, (int64_t)cap, st));
        CK(cub::DeviceScan::ExclusiveSum(nullptr, c, k0, k1, (int64_t)std::max(cap, n_eblocks) + 1, st));
        temp_bytes = std::max(a, std::max(b, c));
        CK(tmp.alloc(reinterpret_cast<unsigned char**>(&temp), temp_bytes));
    }

    for (uint32_t part = 0; part < n_parts; ++part) {
        // K1a: ordered compaction of this partition's windows
        count_part_kernel<<<static_cast<int>(n_eblocks), kEmitThreads, 0, st>>>(ix.planes, n_windows, s, part,
                                                                                 n_parts, bcount);
        CK(cudaGetLastError());
        CK(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, bcount, boff, (int64_t)n_eblocks + 1, st));
        unsigned long long n_p = 0;
        CK(cudaMemsetAsync(bcount + n_eblocks, 0, sizeof(unsigned long long), st));
        CK(cudaMemcpyAsync(&n_p, boff + n_eblocks, sizeof(n_p), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (n_p > cap) {
            err = "index build: partition larger than its buffer";
            free_device_index(&ix);
            return 2;
        }
        ix.n_positions += n_p;
        if (n_p == 0) continue;
        write_part_kernel<<<static_cast<int>(n_eblocks), kEmitThreads, 0, st>>>(ix.planes, n_windows, s, part,
                                                                                 n_parts, boff, k0, v0);
        CK(cudaGetLastError());
        // K1b: stable radix sort by (canon, strand)
        cub::DoubleBuffer<unsigned long long> kb(k0, k1);
        cub::DoubleBuffer<uint32_t> vb(v0, v1);
        CK(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, kb, vb, (int64_t)n_p, 0, end_bit, st));
        // K1c: runs of equal canonical keys (head flags / run ids in the spare buffers)
        uint32_t* head = reinterpret_cast<uint32_t*>(kb.Alternate());
        uint32_t* rid = vb.Alternate();
        head_kernel<<<grid_for(n_p, 256), 256, 0, st>>>(kb.Current(), n_p, s, head);
        CK(cudaGetLastError());
        CK(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, head, rid, (int64_t)n_p, st));
        uint32_t last_head = 0, last_rid = 0;
        CK(cudaMemcpyAsync(&last_head, head + n_p - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&last_rid, rid + n_p - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const uint64_t n_runs = static_cast<uint64_t>(last_rid) + last_head;
        ix.n_keys += n_runs;
        starts_kernel<<<grid_for(n_p, 256), 256, 0, st>>>(head, rid, n_p, run_start);
        CK(cudaGetLastError());
        {
            const uint32_t nv = static_cast<uint32_t>(n_p);
            CK(cudaMemcpyAsync(run_start + n_runs, &nv, 4, cudaMemcpyHostToDevice, st));
        }
        // pool offsets of this partition (head no longer needed: reuse as `need`)
        unsigned long long* need = kb.Alternate();
        pool_need_kernel<<<grid_for(n_runs, 256), 256, 0, st>>>(run_start, n_runs, need);
        CK(cudaGetLastError());
        CK(cudaMemsetAsync(need + n_runs, 0, sizeof(unsigned long long), st));
        CK(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, need, pool_off, (int64_t)n_runs + 1, st));
        unsigned long long part_pool = 0;
        CK(cudaMemcpyAsync(&part_pool, pool_off + n_runs, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (pool_used + part_pool >= 0xffffffffull) {
            err = "position pool exceeds 2^32 entries";
            free_device_index(&ix);
            return 2;
        }
        if (pool_used + part_pool + 1 > pool_cap) {  // grow the pool
            uint64_t ncap = std::max<uint64_t>(pool_cap * 2, pool_used + part_pool + (1 << 20));
            uint32_t* np = nullptr;
            CK(cudaMalloc(&np, ncap * sizeof(uint32_t)));
            CK(cudaMemcpyAsync(np, ix.pool, pool_used * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
            CK(cudaStreamSynchronize(st));
            cudaFree(ix.pool);
            ix.pool = np;
            pool_cap = ncap;
        }
        // K1d
        insert_kernel<<<grid_for(n_runs, 128), 128, 0, st>>>(kb.Current(), vb.Current(), run_start, n_runs,
                                                              pool_off, pool_used, ix.planes, s, ix.table,
                                                              ix.n_slots, ix.pool, d_count);
        CK(cudaGetLastError());
        pool_used += part_pool;
    }
    CK(cudaMemcpyAsync(&ix.n_distinct, d_count, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ix.pool_len = pool_used;
    ix.device_bytes = ix.n_blocks * sizeof(uint4) + ix.n_slots * sizeof(Slot) + pool_cap * sizeof(uint32_t);
    *out = ix;
    return 0;
}

}  // namespace sab
