// align_kernels.cuh -- launch descriptors shared by the host batcher and the
// kernels in align.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/snap_b200.h"
#include "common.cuh"

namespace sab {

// diagnostics: called after each kernel of a seeded launch (align.cu), set by capi.cu
extern thread_local void (*g_timeline_hook)(char tag, cudaStream_t st);

// counters accumulated on the device; first 20 mirror sa_stats
constexpr int kNumStats = 20;

struct AlignLaunch {
    // replica
    const uint4* planes;
    uint64_t glen;
    const Slot* table;
    uint64_t n_slots;
    const uint32_t* pool;
    // reads: read i = bases[offsets[i] - base_off, offsets[i+1] - base_off)
    const char* bases;
    const uint64_t* offsets;
    uint64_t base_off;
    uint32_t n_reads;
    // AlignerParams
    int s, n, dmax_param, c, hmax, bs, force;
    // per-warp layout (units: uint4 blocks / ints / entries)
    int wbr;        // read-plane blocks (fwd and rc each)
    int wbw;        // window staging blocks
    int n_off_cap;  // seed offset slots (ints, multiple of 4)
    int dl_max;     // largest d_limit of the batch
    int f_ints;     // frontier ints (0 when dl_max <= 15)
    int cap;        // candidate list capacity
    int hcap;       // candidate hash slots (power of two)
    int sbw;        // words per read staging buffer (two per warp; 0 = no prefetch)
    int prefetch;   // fast kernel: static striding + cp.async read pipeline
    int dl_prefetch;  // (unused by kernels) reserved
    uint32_t smem_per_warp;
    // outputs
    sa_result* results;
    unsigned long long* stats;  // kNumStats
    unsigned int* cursor;
    unsigned int* overflow_list;
    unsigned int* overflow_count;
    unsigned int* error_flag;
    unsigned long long* error_read;  // atomicMin of the first bad read (absolute index)
    unsigned long long read_base;    // absolute index of read 0 of this launch
    // slow path: process work_list[0..*work_count) with global candidate tables
    // Streaming (batch path, pipelined kernel): one launch covers the whole
    // batch while chunks are still being copied in.  Chunk c (stream_chunk_of:
    // 16 k, 16 k, 32 k, 64 k, then 128 k reads each) is usable once
    // chunk_flag[c] == epoch (written by a stream memory op after its H2D);
    // its bytes sit at bases + offsets[r] + chunk_adj[c]; every finished read
    // bumps chunk_done[c], which releases that chunk's D2H.  Reads longer
    // than lcap are deferred to the end-of-batch pass.  chunk_flag == nullptr:
    // everything is resident (bytes at bases + offsets[r] - base_off).
    const unsigned int* chunk_flag;
    unsigned int* chunk_done;
    const long long* chunk_adj;
    unsigned int epoch;
    int chunk_shift0, chunk_shift;  // stream_chunk_of
    int lcap;
    int f16;  // LV frontier as 16-bit entries (reads < 32 k bases)
    int gw;   // shared-memory LV reads the genome window from global memory (no staging area)
    // long-read layouts with the systolic LV (dl_max >= 256): the read's
    // planes {R, C} live in a per-warp global slot (gplanes + warp id *
    // gplanes_per_warp uint4s) instead of shared memory -- lv_sys touches
    // them once per 64 rows -- so more warps fit per SM (null: shared memory)
    uint4* gplanes;
    uint32_t gplanes_per_warp;
    int bs_shift;  // log2(bucket_size) when it is a power of two, else -1
    // Two-kernel path (seed_kernel + align_kernel<.., kPre>): per read, the
    // seed kernel writes forward then reverse-complement planes
    // (pre_pstride blocks: two halves), every seed record (pre_rstride
    // entries: {flags, count, payload, offset}) and {length, status << 16 |
    // n_eff}; status 0 ok, 1 shorter than s, 2 bad character, 3 longer than
    // the layout (deferred).
    uint4* pre_planes;
    uint4* pre_recs;
    uint2* pre_meta;
    int pre_pstride, pre_rstride;
    // solo_kernel (thread per read) runs between the two when pre_list is set:
    // it finishes the reads it can and lists the others (pre_list[0 ..
    // *pre_list_count), zeroed by the seed kernel) for the align kernel.
    unsigned int* pre_list;
    unsigned int* pre_list_count;
    // Packed input (pack.cpp): when non-null the seed kernel reads the chunk's
    // bases from three bit planes {lo, hi, n} of pk_wpp words each (bit i =
    // base base_off + i) instead of ASCII bytes; lo & n marks a bad character.
    const uint32_t* packed;
    uint64_t pk_wpp;
    // Every read of the chunk has this length (0: use offsets): read r starts
    // at base base_off + r * fixed_len and the offsets are never copied in.
    uint32_t fixed_len;
    const unsigned int* work_list;
    const unsigned int* work_count;
    unsigned char* gscratch;
    uint64_t gscratch_per_warp;
    // pruning batch (align.cu prune_batch): its shared-memory area, the last
    // prune_batch_bytes() of each warp's share, exists
    int pb_on;
    // diagnostics (SA_DEBUG_SOLO): solo-kernel hand-over reasons
    // [0] a seed with too many hits, [1] too many candidates, [2] a long LV
    unsigned int* dbg;
    // seed_kernel probes the first `eager` seeds of each read (0: all); the
    // rest are left as lazy records for the aligner kernels to probe on demand
    int eager;
    // prune queue (align.cu pq_defer / prune_kernel), kPre warp kernel only:
    // pool of pq_cap bytes, byte cursor, records listed in pq_list[0 .. *pq_count)
    // (16-byte units), work cursor for prune_kernel; zeroed by the seed kernel
    unsigned char* pq_pool;
    uint64_t pq_cap;
    unsigned long long* pq_cursor;
    unsigned int* pq_count;
    unsigned int* pq_cursor2;
    unsigned int* pq_list;
    // kPre path: the warp kernel's dynamic read cursor (one listed read per
    // grab), zeroed by the seed kernel; null = static striding
    unsigned int* work_cursor;
};

#ifndef SA_FAST_WARPS
#define SA_FAST_WARPS 8  // warps per block of the align kernels (compile-time: launch bounds)
#endif
#ifndef SA_MIN_BLOCKS
#define SA_MIN_BLOCKS 3  // blocks of SA_FAST_WARPS warps per SM the register budget must allow
#endif
// warps per SM the align kernels' register budget allows
constexpr int kRegWarpsPerSM = SA_FAST_WARPS * SA_MIN_BLOCKS;

// Streamed chunk of read r.  Chunk sizes: 2^first_shift reads for the first
// two chunks, then 2^shift each (both runtime launch fields): short first
// chunks start the kernel early, later ones keep copies efficient.
__host__ __device__ inline uint32_t stream_chunk_of(uint32_t r, int shift0, int shift) {
    const uint32_t head = 2u << shift0;
    if (r < head) return r >> shift0;
    return 2 + ((r - head) >> shift);
}
__host__ __device__ inline uint32_t stream_chunk_begin(uint32_t c, int shift0, int shift) {
    if (c <= 2) return c << shift0;
    return (2u << shift0) + ((c - 2) << shift);
}

// bytes of one candidate table with capacity cap and hcap hash slots
inline uint64_t cand_table_bytes(int cap, int hcap) {
    return static_cast<uint64_t>(cap) * (8 + 8 + 4 + 4) + static_cast<uint64_t>(hcap) * (8 + 4);
}

struct LvLaunch {
    const char* reads;
    const uint64_t* read_off;
    const char* wins;
    const uint64_t* win_off;
    const int32_t* d_limits;
    uint32_t n_pairs;
    int wbr, wbw, f_ints;
    uint32_t smem_per_warp;
    int32_t* out;
    unsigned int* error_flag;
    int bitpar;  // test hook: lv_bitpar for limits <= 15 (set by launch_lv_batch from SA_LV_BITPAR)
    int bitpar_min;  // lv_bitpar_warp from this limit (SA_LV_WARP_BITPAR_MIN test hook)
};

struct LookupLaunch {
    const uint4* planes;
    const Slot* table;
    uint64_t n_slots;
    const uint32_t* pool;
    const char* seeds;
    uint64_t n_seeds;
    int s;
    uint32_t* counts;
    uint64_t* fwd_out;
    uint32_t* n_fwd;
    uint64_t* rc_out;
    uint32_t* n_rc;
    uint32_t cap;
};

void launch_align_fast(const AlignLaunch& a, int grid, int block, cudaStream_t st);
// seed_kernel then the kPre align kernel (a.pre_* set); reads <= 1 kbp
int launch_align_pre(const AlignLaunch& a, int grid, int block, cudaStream_t st);  // kernels launched
void launch_seed(const AlignLaunch& a, cudaStream_t st);                                    // stage 1 only
int launch_align_seeded(const AlignLaunch& a, int grid, int block, cudaStream_t st);      // stage 2 only
void launch_align_slow(const AlignLaunch& a, int grid, int block, cudaStream_t st);
void launch_lv_batch(const LvLaunch& a, int grid, int block, cudaStream_t st);
void launch_lookup(const LookupLaunch& a, cudaStream_t st);
cudaError_t align_fast_occupancy(const AlignLaunch& a, int block, uint32_t smem_bytes, int* blocks_per_sm);
cudaError_t align_set_smem(uint32_t smem_bytes);
uint32_t prune_batch_bytes();
uint32_t prune_kernel_smem_per_warp();  // per warp, appended to the align kernels' shared-memory layout

}  // namespace sab
