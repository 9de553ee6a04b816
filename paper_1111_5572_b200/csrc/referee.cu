// referee.cu -- the exhaustive referee on the GPU.
//
// REF src/eval.cpp:122-306 (OracleIndex, OracleContext, oracle_scan,
// oracle_align): every genome position that can hold the read within d_limit
// edits is verified with bounded_distance.  The candidate set is the
// reference's, exactly: the read (each strand) is cut into d_limit + 1 + #N
// pieces of length L / pieces; any location within d_limit contains one piece
// verbatim at a shift of at most d_limit, so each exact q-gram hit of a piece
// (q = the largest table q <= piece length) contributes the positions
// [x - a - d_limit, x - a + d_limit]; with no usable table every position is a
// candidate.  Candidates are reduced to per-bucket minima (earliest position
// on ties), hits are sorted best-first and, for oracle_align, fed to the same
// BestTracker / classify_confidence as the aligner, in two stages
// (d_limit min(6, full), then full when the cheap stage cannot decide).
//
// GPU layout: q-gram tables (4^q + 1 starts, positions ascending per key)
// built with a CUB sort; per batch of reads, one job per (read, strand):
//   R0 decode      warp/read: forward + reverse-complement read planes
//   R1 count       thread/job: pieces, table, number of candidate intervals
//   R2 intervals   warp/job: (job, lo) keys + hi, CUB radix sort
//   R3 merge       warp/job: disjoint candidate runs, work items of <= 256
//   R4 verify      warp/work item: LV of the read at every position (lv.cuh),
//                  a lane per position (bit-parallel LV) when d_limit <= 15
//   R5 buckets     warp/job: per-bucket minima -> hit keys (dist, pos, dir)
//   R6 sort        CUB segmented sort of each read's hits
//   R7 classify    thread/read: stage decision, BestTracker, classification
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "device_index.h"
#include "host_common.h"
#include "lv.cuh"

using sab::fail_thread;

namespace sab {
namespace {

constexpr int kMaxTables = 4;
constexpr uint32_t kNoDist = 0xffffu;
constexpr uint64_t kSpan = 256;  // positions per verify work item

struct Table {
    int q = 0;
    uint32_t* starts = nullptr;     // 4^q + 1
    uint32_t* positions = nullptr;  // windows without N, ascending per key
};

struct RefView {  // kernel-side view of the referee
    const uint4* planes;
    uint64_t glen;
    int n_tables;
    int q[kMaxTables];
    const uint32_t* starts[kMaxTables];
    const uint32_t* positions[kMaxTables];
};

// ---------------------------------------------------------------- tables

__global__ void qgram_keys_kernel(const uint4* __restrict__ planes, uint64_t n_windows, int q,
                                  uint32_t* __restrict__ keys, uint32_t* __restrict__ pos,
                                  unsigned long long* __restrict__ counts) {
    for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < n_windows;
         p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t lo, hi, n;
        extract32_ldg(planes, p, lo, hi, n);
        uint32_t k = 0xffffffffu;  // windows with N sort last and are dropped
        if (!(n & seed_mask32(q))) {
            k = static_cast<uint32_t>(packed_key(lo, hi, q));
            atomicAdd(counts + k, 1ull);
        }
        keys[p] = k;
        pos[p] = static_cast<uint32_t>(p);
    }
}

__global__ void u64_to_u32_kernel(const unsigned long long* __restrict__ in, uint32_t* __restrict__ out, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<uint32_t>(in[i]);
}

int grid(uint64_t n, int threads) {
    uint64_t g = (n + threads - 1) / threads;
    return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(g, 148ull * 64)));
}

// ---------------------------------------------------------------- batch kernels

struct BatchView {
    const char* bases;
    const uint64_t* offs;
    uint32_t n_reads;
    uint32_t blocks_per_read;  // plane blocks per orientation (incl. the all-N pad)
    uint4* planes;             // [read][dir][blocks]
    uint32_t* n_count;         // N bases per read
    const int32_t* dl;         // d_limit per read
    unsigned int* bad;         // non-ACGTN character seen
};

SA_DEV int base_code(unsigned char c) { return read_code(c); }

// R0: warp per read
__global__ void decode_kernel(BatchView b) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < b.n_reads; r += nw) {
        const char* s = b.bases + b.offs[r];
        const int L = static_cast<int>(b.offs[r + 1] - b.offs[r]);
        uint4* F = b.planes + static_cast<uint64_t>(r) * 2 * b.blocks_per_read;
        uint4* Rc = F + b.blocks_per_read;
        uint32_t nn_total = 0;
        bool bad = false;
        const int nb = (L + 31) / 32;
        for (int blk = 0; blk <= nb; ++blk) {
            const int i = blk * 32 + lane;
            int cf = 4, cr = 4;
            if (i < L) {
                cf = base_code(static_cast<unsigned char>(s[i]));
                const int cs = base_code(static_cast<unsigned char>(s[L - 1 - i]));
                bad |= cf == 5;
                cr = cs >= 4 ? cs : 3 - cs;  // complement (REF genome.cpp:182-200)
                if (cf == 4) ++nn_total;
            }
            const uint32_t flo = __ballot_sync(kLvFull, cf < 4 && (cf & 1)), fhi = __ballot_sync(kLvFull, cf < 4 && (cf & 2));
            const uint32_t fn = __ballot_sync(kLvFull, cf >= 4);
            const uint32_t rlo = __ballot_sync(kLvFull, cr < 4 && (cr & 1)), rhi = __ballot_sync(kLvFull, cr < 4 && (cr & 2));
            const uint32_t rn = __ballot_sync(kLvFull, cr >= 4);
            if (lane == 0) {
                F[blk] = make_uint4(flo, fhi, fn, 0);
                Rc[blk] = make_uint4(rlo, rhi, rn, 0);
            }
        }
        for (int o = 16; o > 0; o >>= 1) nn_total += __shfl_xor_sync(kLvFull, nn_total, o);
        if (__any_sync(kLvFull, bad) && lane == 0) atomicOr(b.bad, 1u);
        if (lane == 0) b.n_count[r] = nn_total;
    }
}

struct JobView {
    uint32_t n_jobs;
    int8_t* table;               // table index, -1 = every position
    int32_t* piece_len;
    int32_t* n_pieces;
    unsigned long long* n_int;   // intervals per job (count pass)
    unsigned long long* int_off; // exclusive scan
};

SA_DEV const uint4* job_planes(const BatchView& b, uint32_t job) {
    return b.planes + static_cast<uint64_t>(job >> 1) * 2 * b.blocks_per_read + (job & 1) * b.blocks_per_read;
}

// q bases of an oriented read at offset a -> packed key; false if any N
SA_DEV bool piece_key(const uint4* R, int a, int q, uint32_t& key) {
    uint32_t lo, hi, n;
    extract32(R, static_cast<uint64_t>(a), lo, hi, n);
    if (n & seed_mask32(q)) return false;
    key = static_cast<uint32_t>(packed_key(lo, hi, q));
    return true;
}

// R1: thread per job (REF eval.cpp:176-205)
__global__ void count_kernel(BatchView b, RefView rv, JobView j) {
    for (uint32_t job = blockIdx.x * blockDim.x + threadIdx.x; job < j.n_jobs; job += gridDim.x * blockDim.x) {
        const uint32_t r = job >> 1;
        const int L = static_cast<int>(b.offs[r + 1] - b.offs[r]);
        const int dl = b.dl[r];
        const int pieces = dl + 1 + static_cast<int>(b.n_count[r]);
        const int plen = L / pieces;
        int t = -1;
        if (plen > 0)
            for (int i = 0; i < rv.n_tables; ++i)
                if (rv.q[i] <= plen) {
                    t = i;
                    break;
                }
        unsigned long long n = 0;
        if (L == 0 || rv.glen == 0) {
            n = 0;
        } else if (t < 0) {
            n = 1;  // every genome position (REF :188-190)
        } else {
            const uint4* R = job_planes(b, job);
            for (int i = 0; i < pieces; ++i) {
                uint32_t key;
                if (!piece_key(R, i * plen, rv.q[t], key)) continue;
                n += rv.starts[t][key + 1] - rv.starts[t][key];
            }
        }
        j.table[job] = static_cast<int8_t>(t);
        j.piece_len[job] = plen;
        j.n_pieces[job] = pieces;
        j.n_int[job] = n;
    }
}

// R2: warp per job: keys (job << 32 | lo), values hi
__global__ void intervals_kernel(BatchView b, RefView rv, JobView j, unsigned long long* __restrict__ ikey,
                                 uint32_t* __restrict__ ihi) {
    const int lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t job = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; job < j.n_jobs; job += nw) {
        if (j.n_int[job] == 0) continue;
        unsigned long long o = j.int_off[job];
        const unsigned long long jk = static_cast<unsigned long long>(job) << 32;
        const int t = j.table[job];
        if (t < 0) {
            if (lane == 0) {
                ikey[o] = jk;
                ihi[o] = static_cast<uint32_t>(rv.glen - 1);
            }
            continue;
        }
        const int dl = b.dl[job >> 1];
        const int plen = j.piece_len[job];
        const uint4* R = job_planes(b, job);
        const int64_t gl = static_cast<int64_t>(rv.glen);
        for (int i = 0; i < j.n_pieces[job]; ++i) {
            uint32_t key;
            if (!piece_key(R, i * plen, rv.q[t], key)) continue;
            const uint32_t s0 = rv.starts[t][key], s1 = rv.starts[t][key + 1];
            const int64_t a = static_cast<int64_t>(i) * plen;
            for (uint32_t h = s0 + lane; h < s1; h += 32) {
                const int64_t center = static_cast<int64_t>(rv.positions[t][h]) - a;
                int64_t lo = center - dl, hi = center + dl;
                if (lo < 0) lo = 0;
                if (hi >= gl) hi = gl - 1;
                // an empty range (hi < lo: the whole window left of 0) keeps
                // its slot as lo = 1, hi = 0; the merge drops it
                const bool empty = hi < lo;
                ikey[o + (h - s0)] = jk | (empty ? 1u : static_cast<uint32_t>(lo));
                ihi[o + (h - s0)] = empty ? 0u : static_cast<uint32_t>(hi);
            }
            o += s1 - s0;
        }
    }
}

struct MergeView {
    unsigned long long* n_cand;   // candidate positions per job
    unsigned long long* n_items;  // verify work items per job
    unsigned long long* n_hitcap; // bound on buckets per job
    unsigned long long* cand_off;
    unsigned long long* item_off;
    unsigned long long* hit_off;  // per job, inside its read's segment
    uint32_t* n_runs;             // merged runs per job (stored in place)
};

// R3: thread per job: merge sorted intervals into disjoint runs (in place)
__global__ void merge_kernel(JobView j, MergeView m, unsigned long long* __restrict__ ikey, uint32_t* __restrict__ ihi,
                             int bucket) {
    for (uint32_t job = blockIdx.x * blockDim.x + threadIdx.x; job < j.n_jobs; job += gridDim.x * blockDim.x) {
        const unsigned long long b0 = j.int_off[job], n = j.n_int[job];
        uint32_t runs = 0;
        unsigned long long cand = 0, items = 0, hitcap = 0;
        bool open = false;
        uint32_t clo = 0, chi = 0;
        auto close = [&]() {
            ikey[b0 + runs] = (ikey[b0] & 0xffffffff00000000ull) | clo;
            ihi[b0 + runs] = chi;
            ++runs;
            const unsigned long long len = static_cast<unsigned long long>(chi) - clo + 1;
            cand += len;
            items += (len + kSpan - 1) / kSpan;
            hitcap += chi / static_cast<uint32_t>(bucket) - clo / static_cast<uint32_t>(bucket) + 1;
        };
        for (unsigned long long i = 0; i < n; ++i) {
            const uint32_t lo = static_cast<uint32_t>(ikey[b0 + i]);
            const uint32_t hi = ihi[b0 + i];
            if (hi < lo) continue;  // empty range
            if (open && static_cast<unsigned long long>(lo) <= static_cast<unsigned long long>(chi) + 1) {
                chi = max(chi, hi);
            } else {
                if (open) close();
                clo = lo;
                chi = hi;
                open = true;
            }
        }
        if (open) close();
        m.n_runs[job] = runs;
        m.n_cand[job] = cand;
        m.n_items[job] = items;
        m.n_hitcap[job] = hitcap;
    }
}

struct Item {
    uint32_t job, lo, hi, pad;
    unsigned long long cand;  // output index of position lo
};

// R3 (warp per job): the same merge, 32 intervals at a time.  Interval i
// opens a run iff its lo is past every earlier hi + 1 (a prefix max carried
// across chunks); a run's hi is the max over its intervals (segmented max).
// Closed runs are written in place at indices no later than the intervals
// they came from, all of which the warp has already loaded.
__global__ void merge_warp_kernel(JobView j, MergeView m, unsigned long long* __restrict__ ikey,
                                  uint32_t* __restrict__ ihi, int bucket) {
    constexpr unsigned kFull = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u, le = lt | (1u << lane);
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t job = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; job < j.n_jobs; job += nw) {
        const unsigned long long b0 = j.int_off[job], n = j.n_int[job];
        const unsigned long long jkey = n ? (ikey[b0] & 0xffffffff00000000ull) : 0;
        uint32_t runs = 0;
        unsigned long long cand = 0, items = 0, hitcap = 0;
        bool open = false;                 // a run is open (carried)
        long long cmax = -2;               // max hi of every interval so far
        uint32_t clo = 0, chi = 0;         // the open run
        auto close_run = [&](uint32_t lo, uint32_t hi, bool mine, unsigned mask) {
            const unsigned before = __popc(mask & lt);
            if (mine) {
                ikey[b0 + runs + before] = jkey | lo;
                ihi[b0 + runs + before] = hi;
            }
            runs += __popc(mask);
            unsigned long long cl = 0, it = 0, hc = 0;
            if (mine) {
                cl = static_cast<unsigned long long>(hi) - lo + 1;
                it = (cl + kSpan - 1) / kSpan;
                hc = hi / static_cast<uint32_t>(bucket) - lo / static_cast<uint32_t>(bucket) + 1;
            }
            for (int o = 16; o > 0; o >>= 1) {
                cl += __shfl_xor_sync(kFull, cl, o);
                it += __shfl_xor_sync(kFull, it, o);
                hc += __shfl_xor_sync(kFull, hc, o);
            }
            cand += cl;
            items += it;
            hitcap += hc;
        };
        for (unsigned long long base = 0; base < n; base += 32) {
            const unsigned long long i = base + lane;
            uint32_t lo = 0, hi = 0;
            bool valid = false;
            if (i < n) {
                lo = static_cast<uint32_t>(ikey[b0 + i]);
                hi = ihi[b0 + i];
                valid = hi >= lo;  // empty ranges are skipped
            }
            __syncwarp();  // every lane has read its interval before any run is written back
            // exclusive prefix max of hi over earlier valid lanes, with the carry
            long long pm = valid ? static_cast<long long>(hi) : -2;
            for (int dd = 1; dd < 32; dd <<= 1) {
                const long long up = __shfl_up_sync(kFull, pm, dd);
                if (lane >= dd && up > pm) pm = up;
            }
            long long excl = __shfl_up_sync(kFull, pm, 1);
            if (lane == 0) excl = -2;
            if (cmax > excl) excl = cmax;
            const unsigned vmask = __ballot_sync(kFull, valid);
            const bool any_before = open || (vmask & lt) != 0u;
            const bool start = valid && (!any_before || static_cast<long long>(lo) > excl + 1);
            const unsigned starts = __ballot_sync(kFull, start);
            // the open run closes where this chunk starts a new one
            if (open && starts != 0u) {
                // its hi grows with the valid intervals before the first start
                const unsigned pre = vmask & ((starts & (0u - starts)) - 1u);
                long long h = (pre >> lane) & 1u ? static_cast<long long>(hi) : -1;
                for (int o = 16; o > 0; o >>= 1) {
                    const long long x = __shfl_xor_sync(kFull, h, o);
                    if (x > h) h = x;
                }
                if (h > static_cast<long long>(chi)) chi = static_cast<uint32_t>(h);
                close_run(clo, chi, lane == 0, 1u);
                open = false;
            }
            // runs started in this chunk: segmented max of hi from each start
            const unsigned sl = starts & le;
            const int seg = sl ? 31 - __clz(sl) : -1;
            long long rh = (valid && seg >= 0) ? static_cast<long long>(hi) : -1;
            for (int dd = 1; dd < 32; dd <<= 1) {
                const long long up = __shfl_up_sync(kFull, rh, dd);
                if (lane >= dd && lane - dd >= seg && seg >= 0 && up > rh) rh = up;
            }
            // a run ends at the last valid lane before the next start; the chunk's last run stays open
            const int last_start = starts ? 31 - __clz(starts) : -1;
            const unsigned after = (lane < 31) ? (starts >> (lane + 1)) : 0u;
            const unsigned next_start_rel = after & (0u - after);  // lowest later start (relative)
            const int nxt = next_start_rel ? lane + 1 + __ffs(next_start_rel) - 1 : 32;
            // the lane just before the next start closes its run (valid lanes only carry hi)
            const bool closes = seg >= 0 && seg != last_start && nxt < 32 && lane == nxt - 1;
            const uint32_t run_lo = __shfl_sync(kFull, lo, seg < 0 ? 0 : seg);
            close_run(run_lo, static_cast<uint32_t>(rh), closes, __ballot_sync(kFull, closes));
            if (last_start >= 0) {  // the last run of the chunk stays open
                const long long h_last = __shfl_sync(kFull, rh, 31);
                clo = __shfl_sync(kFull, lo, last_start);
                chi = static_cast<uint32_t>(h_last);
                open = true;
            } else if (open) {  // no start: every valid interval extends the open run
                long long h = valid ? static_cast<long long>(hi) : -1;
                for (int o = 16; o > 0; o >>= 1) {
                    const long long x = __shfl_xor_sync(kFull, h, o);
                    if (x > h) h = x;
                }
                if (h > static_cast<long long>(chi)) chi = static_cast<uint32_t>(h);
            }
            const long long cm = __shfl_sync(kFull, pm, 31);
            if (cm > cmax) cmax = cm;
        }
        if (open) close_run(clo, chi, lane == 0, 1u);
        if (lane == 0) {
            m.n_runs[job] = runs;
            m.n_cand[job] = cand;
            m.n_items[job] = items;
            m.n_hitcap[job] = hitcap;
        }
    }
}

// R3b: thread per job: verify work items of <= kSpan positions
__global__ void items_kernel(JobView j, MergeView m, const unsigned long long* __restrict__ ikey,
                             const uint32_t* __restrict__ ihi, Item* __restrict__ items) {
    for (uint32_t job = blockIdx.x * blockDim.x + threadIdx.x; job < j.n_jobs; job += gridDim.x * blockDim.x) {
        unsigned long long it = m.item_off[job], c = m.cand_off[job];
        const unsigned long long b0 = j.int_off[job];
        for (uint32_t k = 0; k < m.n_runs[job]; ++k) {
            const uint32_t lo = static_cast<uint32_t>(ikey[b0 + k]), hi = ihi[b0 + k];
            for (unsigned long long p = lo; p <= hi; p += kSpan) {
                const unsigned long long e = p + kSpan - 1 < hi ? p + kSpan - 1 : hi;
                items[it++] = Item{job, static_cast<uint32_t>(p), static_cast<uint32_t>(e), 0, c};
                c += e - p + 1;
            }
        }
    }
}

// R3b (warp per job): the same work items, a lane per run: item and
// candidate offsets by warp prefix sums over 32 runs at a time.
__global__ void items_warp_kernel(JobView j, MergeView m, const unsigned long long* __restrict__ ikey,
                                  const uint32_t* __restrict__ ihi, Item* __restrict__ items) {
    constexpr unsigned kFull = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t job = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; job < j.n_jobs; job += nw) {
        unsigned long long it = m.item_off[job], c = m.cand_off[job];
        const unsigned long long b0 = j.int_off[job];
        const uint32_t nr = m.n_runs[job];
        for (uint32_t k0 = 0; k0 < nr; k0 += 32) {
            const uint32_t k = k0 + lane;
            uint32_t lo = 0, hi = 0;
            unsigned long long len = 0, nit = 0;
            if (k < nr) {
                lo = static_cast<uint32_t>(ikey[b0 + k]);
                hi = ihi[b0 + k];
                len = static_cast<unsigned long long>(hi) - lo + 1;
                nit = (len + kSpan - 1) / kSpan;
            }
            unsigned long long si = nit, sc = len;  // inclusive prefix sums
            for (int dd = 1; dd < 32; dd <<= 1) {
                const unsigned long long ui = __shfl_up_sync(kFull, si, dd), uc = __shfl_up_sync(kFull, sc, dd);
                if (lane >= dd) {
                    si += ui;
                    sc += uc;
                }
            }
            unsigned long long my_it = it + si - nit, my_c = c + sc - len;
            for (unsigned long long p = lo; k < nr && p <= hi; p += kSpan) {
                const unsigned long long e = p + kSpan - 1 < hi ? p + kSpan - 1 : hi;
                items[my_it++] = Item{job, static_cast<uint32_t>(p), static_cast<uint32_t>(e), 0, my_c};
                my_c += e - p + 1;
            }
            it += __shfl_sync(kFull, si, 31);
            c += __shfl_sync(kFull, sc, 31);
        }
    }
}

// R4: warp per work item: bounded_distance at every position of the item.
// kBit (every d_limit <= 15): lane l verifies positions lo + l, lo + l + 32,
// ... with the banded bit-parallel LV (lv.cuh lv_bitpar) -- the same read and
// limit for the whole item, so the warp runs in lock step, and a position far
// from the read costs m + d_limit column steps instead of d_limit + 1 full
// wavefront iterations.  Otherwise the warp runs the wavefront LV position by
// position (lanes = diagonals).
template <bool kReg, bool kBit = false>
__global__ void verify_kernel(BatchView b, RefView rv, const Item* __restrict__ items, unsigned long long n_items,
                              uint16_t* __restrict__ dist, int f_ints) {
    extern __shared__ int smem_f[];
    const int lane = threadIdx.x & 31;
    int* F = smem_f + (threadIdx.x >> 5) * f_ints;
    const unsigned long long nw = (static_cast<unsigned long long>(gridDim.x) * blockDim.x) >> 5;
    for (unsigned long long w = (blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x) >> 5;
         w < n_items; w += nw) {
        const Item it = items[w];
        const uint32_t r = it.job >> 1;
        const int L = static_cast<int>(b.offs[r + 1] - b.offs[r]);
        const int dl = b.dl[r];
        const uint4* R = job_planes(b, it.job);
        uint32_t cells = 0;
        if (kBit) {
            for (uint32_t p0 = it.lo; p0 <= it.hi; p0 += 32) {
                const uint32_t p = p0 + lane;
                if (p <= it.hi) {
                    const uint64_t rem = rv.glen - p;  // REF eval.cpp:223-225
                    const uint64_t want = static_cast<uint64_t>(L) + static_cast<uint64_t>(dl);
                    const int wlen = static_cast<int>(want < rem ? want : rem);
                    const int d = lv_bitpar(R, static_cast<int>(b.blocks_per_read), L, rv.planes, p, wlen, dl, cells);
                    dist[it.cand + (p - it.lo)] = d < 0 ? kNoDist : static_cast<uint16_t>(d);
                }
                if (p0 + 32 < p0) break;  // 32-bit wrap guard
            }
            continue;
        }
        for (uint32_t p = it.lo;; ++p) {
            // REF eval.cpp:223-225: window = substring(p, L + d_limit)
            const uint64_t rem = rv.glen - p;
            const uint64_t want = static_cast<uint64_t>(L) + static_cast<uint64_t>(dl);
            const int wlen = static_cast<int>(want < rem ? want : rem);
            int d;
            if (kReg) d = lv_warp_reg(R, L, rv.planes, p, wlen, dl, lane, cells);
            else d = lv_warp_smem(R, L, rv.planes, p, wlen, dl, F, lane, cells);
            if (lane == 0) dist[it.cand + (p - it.lo)] = d < 0 ? kNoDist : static_cast<uint16_t>(d);
            if (p == it.hi) break;
        }
    }
}

// R5 (warp per job): the same per-bucket minima, 32 candidate positions at a
// time.  Positions ascend within a job, so a bucket is a contiguous segment;
// each chunk takes a segmented min-scan of (distance << 32 | position) -- the
// minimum is the smallest distance, earliest position on ties, as the
// sequential `d < best` keeps -- merged with the bucket still open from the
// previous chunk.  Closed buckets with a hit are written in order (ballot
// prefix); the last segment of a chunk stays open.  Same output as
// bucket_kernel; the serial pass was 76% of the referee's GPU time.
__global__ void bucket_warp_kernel(JobView j, MergeView m, const unsigned long long* __restrict__ ikey,
                                   const uint32_t* __restrict__ ihi, const uint16_t* __restrict__ dist, int bucket,
                                   unsigned long long* __restrict__ hits, uint32_t* __restrict__ n_hits) {
    constexpr unsigned kFull = 0xffffffffu;
    constexpr unsigned long long kNone = ~0ull;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u, le = lt | (1u << lane);
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t job = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; job < j.n_jobs; job += nw) {
        const unsigned long long b0 = j.int_off[job];
        unsigned long long c = m.cand_off[job], o = m.hit_off[job];
        const unsigned long long dir = job & 1;
        long long open_b = -1;               // bucket of the open segment
        unsigned long long open_best = kNone;  // its minimum so far
        uint32_t cnt = 0;
        auto emit = [&](unsigned long long key, bool mine, unsigned mask) {
            // key = d << 32 | p  ->  hit = d << 33 | p << 1 | dir
            const unsigned before = __popc(mask & lt);
            if (mine) hits[o + before] = ((key >> 32) << 33) | ((key & 0xffffffffull) << 1) | dir;
            o += __popc(mask);
            cnt += __popc(mask);
        };
        for (uint32_t k = 0; k < m.n_runs[job]; ++k) {
            const uint32_t lo = static_cast<uint32_t>(ikey[b0 + k]), hi = ihi[b0 + k];
            for (unsigned long long base = lo; base <= hi; base += 32) {
                const unsigned long long p = base + lane;
                const bool valid = p <= hi;
                const long long bk = valid ? static_cast<long long>(p / static_cast<unsigned long long>(bucket)) : -2;
                unsigned long long key = kNone;
                if (valid) {
                    const uint32_t d = dist[c + (p - base)];
                    if (d != kNoDist) key = (static_cast<unsigned long long>(d) << 32) | p;
                }
                const long long bk_prev = __shfl_up_sync(kFull, bk, 1);
                const bool head = valid && (lane == 0 ? bk != open_b : bk != bk_prev);
                const unsigned heads = __ballot_sync(kFull, head);
                const unsigned vmask = __ballot_sync(kFull, valid);
                // a chunk that starts a new bucket closes the open one first
                if ((heads & 1u) && open_b >= 0) emit(open_best, lane == 0 && open_best != kNone,
                                                       __ballot_sync(kFull, lane == 0 && open_best != kNone));
                const unsigned hl = heads & le;
                const int seg = hl ? 31 - __clz(hl) : -1;  // -1: continues the open bucket
                for (int dd = 1; dd < 32; dd <<= 1) {
                    const unsigned long long up = __shfl_up_sync(kFull, key, dd);
                    if (lane - dd >= seg && lane >= dd && up < key) key = up;
                }
                if (valid && seg < 0 && open_best < key) key = open_best;
                // tails: last lane of each segment; the chunk's final segment stays open
                const int last = 31 - __clz(vmask);
                const bool tail = valid && lane != last && ((heads >> (lane + 1)) & 1u);
                const bool out = tail && key != kNone;
                emit(key, out, __ballot_sync(kFull, out));
                open_best = __shfl_sync(kFull, key, last);
                open_b = __shfl_sync(kFull, bk, last);
                c += static_cast<unsigned long long>(__popc(vmask));
            }
        }
        if (open_b >= 0 && open_best != kNone) emit(open_best, lane == 0, 1u);
        if (lane == 0) n_hits[job] = cnt;
    }
}

// R5: thread per job: per-bucket minima (REF eval.cpp:207-232) -> hit keys
// (distance << 33 | position << 1 | direction), sorted later per read
__global__ void bucket_kernel(JobView j, MergeView m, const unsigned long long* __restrict__ ikey,
                              const uint32_t* __restrict__ ihi, const uint16_t* __restrict__ dist, int bucket,
                              unsigned long long* __restrict__ hits, uint32_t* __restrict__ n_hits) {
    for (uint32_t job = blockIdx.x * blockDim.x + threadIdx.x; job < j.n_jobs; job += gridDim.x * blockDim.x) {
        const unsigned long long b0 = j.int_off[job];
        unsigned long long c = m.cand_off[job], o = m.hit_off[job];
        const unsigned long long dir = job & 1;
        long long open_b = -1;
        uint32_t best = kNoDist, best_p = 0, cnt = 0;
        for (uint32_t k = 0; k < m.n_runs[job]; ++k) {
            const uint32_t lo = static_cast<uint32_t>(ikey[b0 + k]), hi = ihi[b0 + k];
            for (unsigned long long p = lo; p <= hi; ++p, ++c) {
                const long long bk = static_cast<long long>(p / static_cast<unsigned long long>(bucket));
                if (bk != open_b) {
                    if (open_b >= 0 && best != kNoDist) {
                        hits[o++] = (static_cast<unsigned long long>(best) << 33) |
                                    (static_cast<unsigned long long>(best_p) << 1) | dir;
                        ++cnt;
                    }
                    open_b = bk;
                    best = kNoDist;
                }
                const uint32_t d = dist[c];
                if (d != kNoDist && d < best) {
                    best = d;
                    best_p = static_cast<uint32_t>(p);
                }
            }
        }
        if (open_b >= 0 && best != kNoDist) {
            hits[o++] = (static_cast<unsigned long long>(best) << 33) | (static_cast<unsigned long long>(best_p) << 1) |
                        dir;
            ++cnt;
        }
        n_hits[job] = cnt;
    }
}

// R7: thread per read: REF eval.cpp:270-306 stage logic + BestTracker
// (aligner.cpp:87-114) + classify_confidence (aligner.cpp:81-85).
// outcome: 0 = decided (result written), 1 = escalate to the full limit
__global__ void classify_kernel(BatchView b, const unsigned long long* __restrict__ hits,
                                const unsigned long long* __restrict__ seg_off, const uint32_t* __restrict__ n_hits,
                                const int32_t* __restrict__ dmax, const uint8_t* __restrict__ final_stage, int c,
                                int bucket, sa_result* __restrict__ res, uint8_t* __restrict__ outcome) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < b.n_reads; r += gridDim.x * blockDim.x) {
        const unsigned long long* h = hits + seg_off[r];
        const uint32_t n = n_hits[2 * r] + n_hits[2 * r + 1];
        sa_result out;
        out.position = 0;
        out.distance = -1;
        out.gap = 0;
        out.kind = SA_NOT_FOUND;
        out.has_position = 0;
        out.direction = 0;
        for (int i = 0; i < 5; ++i) out.reserved[i] = 0;
        const int dl = b.dl[r];
        if (n == 0) {
            outcome[r] = final_stage[r] ? 0 : 1;
            res[r] = out;
            continue;
        }
        if (!final_stage[r] && static_cast<int>(h[0] >> 33) + c - 1 > dl) {
            outcome[r] = 1;
            res[r] = out;
            continue;
        }
        int d_best = kInfDistance, d_second = kInfDistance, best_dir = 0;
        uint64_t best_pos = 0;
        for (uint32_t i = 0; i < n; ++i) {
            const int d = static_cast<int>(h[i] >> 33);
            const uint64_t pos = (h[i] >> 1) & 0xffffffffull;
            const int dir = static_cast<int>(h[i] & 1);
            if (d_best < kInfDistance && dir == best_dir) {
                const uint64_t delta = pos > best_pos ? pos - best_pos : best_pos - pos;
                if (delta <= static_cast<uint64_t>(bucket)) {
                    if (d < d_best) {
                        d_best = d;
                        best_pos = pos;
                    }
                    continue;
                }
            }
            if (d < d_best) {
                d_second = d_best;
                d_best = d;
                best_pos = pos;
                best_dir = dir;
            } else if (d < d_second) {
                d_second = d;
            }
        }
        const int d_max = dmax[r];
        int kind = SA_NOT_FOUND;
        if (d_best <= d_max && d_second >= d_best + c) kind = SA_SINGLE_HIT;
        else if (d_best <= d_max) kind = SA_MULTIPLE_HITS;
        out.kind = static_cast<uint8_t>(kind);
        if (kind != SA_NOT_FOUND && d_best <= d_max) {
            out.has_position = 1;
            out.position = best_pos;
            out.direction = static_cast<uint8_t>(best_dir);
            out.distance = d_best;
            out.gap = d_second >= kInfDistance ? kGapCap : min(d_second - d_best, kGapCap);
        }
        res[r] = out;
        outcome[r] = 0;
    }
}

}  // namespace
}  // namespace sab

// ---------------------------------------------------------------- host side

struct sa_referee {
    int device = 0;
    cudaStream_t st = nullptr;
    uint4* planes = nullptr;
    uint64_t glen = 0;
    std::vector<sab::Table> tables;  // descending q (REF eval.cpp:155-165)
    std::string err;
    ~sa_referee() {
        cudaSetDevice(device);
        for (auto& t : tables) {
            cudaFree(t.starts);
            cudaFree(t.positions);
        }
        if (planes) cudaFree(planes);
        if (st) cudaStreamDestroy(st);
    }
    sab::RefView view() const {
        sab::RefView v{};
        v.planes = planes;
        v.glen = glen;
        v.n_tables = static_cast<int>(tables.size());
        for (size_t i = 0; i < tables.size(); ++i) {
            v.q[i] = tables[i].q;
            v.starts[i] = tables[i].starts;
            v.positions[i] = tables[i].positions;
        }
        return v;
    }
};

namespace {

struct DevBufs {  // freed on scope exit
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
    ~DevBufs() {
        for (void* q : p) cudaFree(q);
    }
};

#define RF_TRY(x)                                                                                  \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess) return fail_thread(SA_ERUNTIME, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// OracleIndex (REF eval.cpp:122-150) for one q on the GPU
int build_table(sa_referee& rf, int q, sab::Table& t) {
    t.q = q;
    const uint64_t n_keys = 1ull << (2 * q);
    const uint64_t n_windows = rf.glen >= static_cast<uint64_t>(q) ? rf.glen - q + 1 : 0;
    RF_TRY(cudaMalloc(&t.starts, (n_keys + 1) * sizeof(uint32_t)));
    DevBufs b;
    unsigned long long* counts = nullptr;
    RF_TRY(b.alloc(&counts, n_keys + 1));
    RF_TRY(cudaMemsetAsync(counts, 0, (n_keys + 1) * sizeof(unsigned long long), rf.st));
    uint32_t *k0 = nullptr, *k1 = nullptr, *v0 = nullptr, *v1 = nullptr;
    RF_TRY(b.alloc(&k0, n_windows));
    RF_TRY(b.alloc(&k1, n_windows));
    RF_TRY(b.alloc(&v0, n_windows));
    RF_TRY(b.alloc(&v1, n_windows));
    if (n_windows)
        sab::qgram_keys_kernel<<<sab::grid(n_windows, 256), 256, 0, rf.st>>>(rf.planes, n_windows, q, k0, v0, counts);
    RF_TRY(cudaGetLastError());
    // starts = exclusive scan of counts (REF :138)
    unsigned long long* scanned = nullptr;
    RF_TRY(b.alloc(&scanned, n_keys + 1));
    size_t tb = 0;
    RF_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, scanned, static_cast<int64_t>(n_keys + 1), rf.st));
    unsigned char* temp = nullptr;
    size_t tb2 = 0;
    cub::DoubleBuffer<uint32_t> kb(k0, k1), vb(v0, v1);
    RF_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb2, kb, vb, static_cast<int64_t>(n_windows), 0, 32, rf.st));
    RF_TRY(b.alloc(&temp, std::max(tb, tb2)));
    RF_TRY(cub::DeviceScan::ExclusiveSum(temp, tb, counts, scanned, static_cast<int64_t>(n_keys + 1), rf.st));
    sab::u64_to_u32_kernel<<<sab::grid(n_keys + 1, 256), 256, 0, rf.st>>>(scanned, t.starts, n_keys + 1);
    RF_TRY(cudaGetLastError());
    unsigned long long total = 0;
    RF_TRY(cudaMemcpyAsync(&total, scanned + n_keys, sizeof(total), cudaMemcpyDeviceToHost, rf.st));
    // positions ascending per key: stable sort of (key, position) in window order
    size_t tsz = std::max(tb, tb2);
    if (n_windows)
        RF_TRY(cub::DeviceRadixSort::SortPairs(temp, tsz, kb, vb, static_cast<int64_t>(n_windows), 0, 32, rf.st));
    RF_TRY(cudaStreamSynchronize(rf.st));
    RF_TRY(cudaMalloc(&t.positions, std::max<uint64_t>(total, 1) * sizeof(uint32_t)));
    RF_TRY(cudaMemcpyAsync(t.positions, vb.Current(), total * sizeof(uint32_t), cudaMemcpyDeviceToDevice, rf.st));
    RF_TRY(cudaStreamSynchronize(rf.st));
    return SA_OK;
}

// One stage over a batch of reads: per-read d_limit / d_max / final flags.
// results/outcome are host arrays of n_reads; hits_out (nullable) receives
// each read's sorted hit keys for sa_referee_scan.
int run_batch(sa_referee& rf, const char* bases, const uint64_t* offs, uint32_t n_reads, const int32_t* dl,
              const int32_t* dmax, const uint8_t* final_stage, int c, int bucket, sa_result* results,
              uint8_t* outcome, std::vector<std::vector<unsigned long long>>* hits_out) {
    using namespace sab;
    if (n_reads == 0) return SA_OK;
    DevBufs B;
    cudaStream_t st = rf.st;
    const uint64_t nbytes = offs[n_reads] - offs[0];
    uint64_t Lmax = 0;
    for (uint32_t i = 0; i < n_reads; ++i) Lmax = std::max(Lmax, offs[i + 1] - offs[i]);
    int dlmax = 0;
    for (uint32_t i = 0; i < n_reads; ++i) dlmax = std::max(dlmax, dl[i]);
    char* d_bases = nullptr;
    uint64_t* d_offs = nullptr;
    RF_TRY(B.alloc(&d_bases, nbytes + 8));
    RF_TRY(B.alloc(&d_offs, n_reads + 1));
    std::vector<uint64_t> rel(n_reads + 1);
    for (uint32_t i = 0; i <= n_reads; ++i) rel[i] = offs[i] - offs[0];
    RF_TRY(cudaMemcpyAsync(d_bases, bases + offs[0], nbytes, cudaMemcpyHostToDevice, st));
    RF_TRY(cudaMemcpyAsync(d_offs, rel.data(), (n_reads + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    BatchView bv{};
    bv.bases = d_bases;
    bv.offs = d_offs;
    bv.n_reads = n_reads;
    bv.blocks_per_read = static_cast<uint32_t>((Lmax + 31) / 32 + 2);
    RF_TRY(B.alloc(&bv.planes, static_cast<uint64_t>(n_reads) * 2 * bv.blocks_per_read));
    RF_TRY(B.alloc(&bv.n_count, n_reads));
    int32_t *d_dl = nullptr, *d_dmax = nullptr;
    uint8_t *d_final = nullptr, *d_outcome = nullptr;
    RF_TRY(B.alloc(&d_dl, n_reads));
    RF_TRY(B.alloc(&d_dmax, n_reads));
    RF_TRY(B.alloc(&d_final, n_reads));
    RF_TRY(B.alloc(&d_outcome, n_reads));
    RF_TRY(cudaMemcpyAsync(d_dl, dl, n_reads * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    RF_TRY(cudaMemcpyAsync(d_dmax, dmax, n_reads * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    RF_TRY(cudaMemcpyAsync(d_final, final_stage, n_reads, cudaMemcpyHostToDevice, st));
    bv.dl = d_dl;
    RF_TRY(B.alloc(&bv.bad, 1));
    RF_TRY(cudaMemsetAsync(bv.bad, 0, sizeof(unsigned int), st));
    decode_kernel<<<grid(static_cast<uint64_t>(n_reads) * 32, 256), 256, 0, st>>>(bv);
    RF_TRY(cudaGetLastError());
    unsigned int bad = 0;
    RF_TRY(cudaMemcpyAsync(&bad, bv.bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
    RF_TRY(cudaStreamSynchronize(st));
    if (bad) return fail_thread(SA_EINVAL, "reverse_complement: non-base character");  // REF genome.cpp:194-195

    const RefView rv = rf.view();
    JobView jv{};
    jv.n_jobs = 2 * n_reads;
    RF_TRY(B.alloc(&jv.table, jv.n_jobs));
    RF_TRY(B.alloc(&jv.piece_len, jv.n_jobs));
    RF_TRY(B.alloc(&jv.n_pieces, jv.n_jobs));
    RF_TRY(B.alloc(&jv.n_int, jv.n_jobs + 1));
    RF_TRY(B.alloc(&jv.int_off, jv.n_jobs + 1));
    count_kernel<<<grid(jv.n_jobs, 128), 128, 0, st>>>(bv, rv, jv);
    RF_TRY(cudaGetLastError());
    RF_TRY(cudaMemsetAsync(jv.n_int + jv.n_jobs, 0, sizeof(unsigned long long), st));
    size_t tbytes = 0;
    RF_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tbytes, jv.n_int, jv.int_off, static_cast<int64_t>(jv.n_jobs + 1), st));
    void* tmp = nullptr;
    RF_TRY(cudaMalloc(&tmp, tbytes));
    B.p.push_back(tmp);
    RF_TRY(cub::DeviceScan::ExclusiveSum(tmp, tbytes, jv.n_int, jv.int_off, static_cast<int64_t>(jv.n_jobs + 1), st));
    unsigned long long n_int = 0;
    RF_TRY(cudaMemcpyAsync(&n_int, jv.int_off + jv.n_jobs, sizeof(n_int), cudaMemcpyDeviceToHost, st));
    RF_TRY(cudaStreamSynchronize(st));

    unsigned long long *ik0 = nullptr, *ik1 = nullptr;
    uint32_t *ih0 = nullptr, *ih1 = nullptr;
    RF_TRY(B.alloc(&ik0, n_int));
    RF_TRY(B.alloc(&ik1, n_int));
    RF_TRY(B.alloc(&ih0, n_int));
    RF_TRY(B.alloc(&ih1, n_int));
    intervals_kernel<<<grid(static_cast<uint64_t>(jv.n_jobs) * 32, 256), 256, 0, st>>>(bv, rv, jv, ik0, ih0);
    RF_TRY(cudaGetLastError());
    int job_bits = 1;
    while ((1ull << job_bits) < jv.n_jobs) ++job_bits;
    cub::DoubleBuffer<unsigned long long> kb(ik0, ik1);
    cub::DoubleBuffer<uint32_t> vb(ih0, ih1);
    size_t sb = 0;
    RF_TRY(cub::DeviceRadixSort::SortPairs(nullptr, sb, kb, vb, static_cast<int64_t>(n_int), 0, 32 + job_bits, st));
    void* stmp = nullptr;
    RF_TRY(cudaMalloc(&stmp, std::max<size_t>(sb, 1)));
    B.p.push_back(stmp);
    if (n_int) RF_TRY(cub::DeviceRadixSort::SortPairs(stmp, sb, kb, vb, static_cast<int64_t>(n_int), 0, 32 + job_bits, st));
    unsigned long long* ikey = kb.Current();
    uint32_t* ihi = vb.Current();

    MergeView mv{};
    RF_TRY(B.alloc(&mv.n_cand, jv.n_jobs + 1));
    RF_TRY(B.alloc(&mv.n_items, jv.n_jobs + 1));
    RF_TRY(B.alloc(&mv.n_hitcap, jv.n_jobs + 1));
    RF_TRY(B.alloc(&mv.cand_off, jv.n_jobs + 1));
    RF_TRY(B.alloc(&mv.item_off, jv.n_jobs + 1));
    RF_TRY(B.alloc(&mv.hit_off, jv.n_jobs + 1));
    RF_TRY(B.alloc(&mv.n_runs, jv.n_jobs));
    if (getenv("SA_REF_MERGE_SERIAL") == nullptr) {  // A/B switch: the thread-per-job pass
        const uint64_t wg = std::min<uint64_t>((jv.n_jobs + 7) / 8, 148ull * 64);
        merge_warp_kernel<<<static_cast<int>(std::max<uint64_t>(wg, 1)), 256, 0, st>>>(jv, mv, ikey, ihi, bucket);
    } else {
        merge_kernel<<<grid(jv.n_jobs, 128), 128, 0, st>>>(jv, mv, ikey, ihi, bucket);
    }
    RF_TRY(cudaGetLastError());
    RF_TRY(cudaMemsetAsync(mv.n_cand + jv.n_jobs, 0, sizeof(unsigned long long), st));
    RF_TRY(cudaMemsetAsync(mv.n_items + jv.n_jobs, 0, sizeof(unsigned long long), st));
    RF_TRY(cudaMemsetAsync(mv.n_hitcap + jv.n_jobs, 0, sizeof(unsigned long long), st));
    RF_TRY(cub::DeviceScan::ExclusiveSum(tmp, tbytes, mv.n_cand, mv.cand_off, static_cast<int64_t>(jv.n_jobs + 1), st));
    RF_TRY(cub::DeviceScan::ExclusiveSum(tmp, tbytes, mv.n_items, mv.item_off, static_cast<int64_t>(jv.n_jobs + 1), st));
    RF_TRY(cub::DeviceScan::ExclusiveSum(tmp, tbytes, mv.n_hitcap, mv.hit_off, static_cast<int64_t>(jv.n_jobs + 1), st));
    unsigned long long tot[3] = {};
    RF_TRY(cudaMemcpyAsync(&tot[0], mv.cand_off + jv.n_jobs, 8, cudaMemcpyDeviceToHost, st));
    RF_TRY(cudaMemcpyAsync(&tot[1], mv.item_off + jv.n_jobs, 8, cudaMemcpyDeviceToHost, st));
    RF_TRY(cudaMemcpyAsync(&tot[2], mv.hit_off + jv.n_jobs, 8, cudaMemcpyDeviceToHost, st));
    RF_TRY(cudaStreamSynchronize(st));
    Item* items = nullptr;
    uint16_t* dist = nullptr;
    RF_TRY(B.alloc(&items, tot[1]));
    RF_TRY(B.alloc(&dist, tot[0]));
    if (getenv("SA_REF_MERGE_SERIAL") == nullptr) {  // (same A/B switch as the merge)
        const uint64_t wg = std::min<uint64_t>((jv.n_jobs + 7) / 8, 148ull * 64);
        items_warp_kernel<<<static_cast<int>(std::max<uint64_t>(wg, 1)), 256, 0, st>>>(jv, mv, ikey, ihi, items);
    } else {
        items_kernel<<<grid(jv.n_jobs, 128), 128, 0, st>>>(jv, mv, ikey, ihi, items);
    }
    RF_TRY(cudaGetLastError());
    if (tot[1]) {
        const int f_ints = dlmax > 15 ? 2 * (2 * dlmax + 3) : 0;
        int warps = 8;
        if (f_ints) warps = std::max(1, std::min(8, static_cast<int>((200 * 1024) / (f_ints * 4))));
        const uint64_t want = std::min<uint64_t>(tot[1], 148ull * 64);
        const int g = static_cast<int>((want + warps - 1) / warps);
        const size_t smem = static_cast<size_t>(f_ints) * 4 * warps;
        if (f_ints) {
            RF_TRY(cudaFuncSetAttribute(verify_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
            verify_kernel<false><<<g, 32 * warps, smem, st>>>(bv, rv, items, tot[1], dist, f_ints);
        } else if (getenv("SA_REF_WAVEFRONT") == nullptr) {  // A/B switch: the wavefront LV
            verify_kernel<true, true><<<g, 32 * warps, 0, st>>>(bv, rv, items, tot[1], dist, 0);
        } else {
            verify_kernel<true><<<g, 32 * warps, 0, st>>>(bv, rv, items, tot[1], dist, 0);
        }
        RF_TRY(cudaGetLastError());
    }
    // hits: each read's segment = its two jobs' bounds; unused slots sort last
    unsigned long long* hits = nullptr;
    uint32_t* n_hits = nullptr;
    RF_TRY(B.alloc(&hits, tot[2]));
    RF_TRY(B.alloc(&n_hits, jv.n_jobs));
    RF_TRY(cudaMemsetAsync(hits, 0xff, std::max<unsigned long long>(tot[2], 1) * 8, st));
    if (getenv("SA_REF_BUCKET_SERIAL") == nullptr) {  // A/B switch: the thread-per-job pass
        const uint64_t wg = std::min<uint64_t>((jv.n_jobs + 7) / 8, 148ull * 64);
        bucket_warp_kernel<<<static_cast<int>(std::max<uint64_t>(wg, 1)), 256, 0, st>>>(jv, mv, ikey, ihi, dist, bucket,
                                                                                       hits, n_hits);
    } else {
        bucket_kernel<<<grid(jv.n_jobs, 128), 128, 0, st>>>(jv, mv, ikey, ihi, dist, bucket, hits, n_hits);
    }
    RF_TRY(cudaGetLastError());
    // read segment offsets = job hit offsets of even jobs (+ the total)
    std::vector<unsigned long long> job_off(jv.n_jobs + 1);
    RF_TRY(cudaMemcpyAsync(job_off.data(), mv.hit_off, (jv.n_jobs + 1) * 8, cudaMemcpyDeviceToHost, st));
    RF_TRY(cudaStreamSynchronize(st));
    std::vector<unsigned long long> seg(n_reads + 1);
    for (uint32_t r = 0; r < n_reads; ++r) seg[r] = job_off[2 * r];
    seg[n_reads] = job_off[jv.n_jobs];
    unsigned long long* d_seg = nullptr;
    RF_TRY(B.alloc(&d_seg, n_reads + 1));
    RF_TRY(cudaMemcpyAsync(d_seg, seg.data(), (n_reads + 1) * 8, cudaMemcpyHostToDevice, st));
    unsigned long long* hits_sorted = nullptr;
    RF_TRY(B.alloc(&hits_sorted, tot[2]));
    if (tot[2]) {
        size_t ssb = 0;
        RF_TRY(cub::DeviceSegmentedSort::SortKeys(nullptr, ssb, hits, hits_sorted, static_cast<int64_t>(tot[2]),
                                                  static_cast<int64_t>(n_reads), d_seg, d_seg + 1, st));
        void* sst = nullptr;
        RF_TRY(cudaMalloc(&sst, std::max<size_t>(ssb, 1)));
        B.p.push_back(sst);
        RF_TRY(cub::DeviceSegmentedSort::SortKeys(sst, ssb, hits, hits_sorted, static_cast<int64_t>(tot[2]),
                                                  static_cast<int64_t>(n_reads), d_seg, d_seg + 1, st));
    }
    sa_result* d_res = nullptr;
    RF_TRY(B.alloc(&d_res, n_reads));
    classify_kernel<<<grid(n_reads, 128), 128, 0, st>>>(bv, hits_sorted, d_seg, n_hits, d_dmax, d_final, c, bucket,
                                                         d_res, d_outcome);
    RF_TRY(cudaGetLastError());
    RF_TRY(cudaMemcpyAsync(results, d_res, n_reads * sizeof(sa_result), cudaMemcpyDeviceToHost, st));
    RF_TRY(cudaMemcpyAsync(outcome, d_outcome, n_reads, cudaMemcpyDeviceToHost, st));
    if (hits_out) {
        std::vector<uint32_t> nh(jv.n_jobs);
        std::vector<unsigned long long> all(tot[2]);
        RF_TRY(cudaMemcpyAsync(nh.data(), n_hits, jv.n_jobs * 4, cudaMemcpyDeviceToHost, st));
        RF_TRY(cudaMemcpyAsync(all.data(), hits_sorted, tot[2] * 8, cudaMemcpyDeviceToHost, st));
        RF_TRY(cudaStreamSynchronize(st));
        hits_out->resize(n_reads);
        for (uint32_t r = 0; r < n_reads; ++r)
            (*hits_out)[r].assign(all.begin() + static_cast<long>(seg[r]),
                                  all.begin() + static_cast<long>(seg[r] + nh[2 * r] + nh[2 * r + 1]));
    }
    RF_TRY(cudaStreamSynchronize(st));
    return SA_OK;
}

int effective_dmax(const sa_params* p, uint64_t L) {  // REF aligner.cpp:26-29
    return p->max_distance >= 0 ? p->max_distance : static_cast<int>((12 * L + 99) / 100);
}

// reads per GPU batch: bounded so candidate arrays stay modest
constexpr uint32_t kBatchReads = 1u << 15;

}  // namespace

extern "C" {

int sa_referee_create(const sa_genome* g, int32_t device, sa_referee** out) {
    if (!g || !out) return fail_thread(SA_EINVAL, "null argument");
    *out = nullptr;
    if (g->length > 0xffffffffull - 64) return fail_thread(SA_EINVAL, "genome longer than 2^32 - 64 bases");
    auto rf = std::make_unique<sa_referee>();
    rf->device = device;
    RF_TRY(cudaSetDevice(device));
    RF_TRY(cudaStreamCreateWithFlags(&rf->st, cudaStreamNonBlocking));
    rf->glen = g->length;
    if (rf->glen > 0) {
        std::string err;
        if (sab::upload_planes(g->packed.data(), g->packed.size(), g->nmask.data(), g->nmask.size(), g->length,
                               rf->st, &rf->planes, err))
            return fail_thread(SA_ERUNTIME, err);
    }
    // OracleContext (REF eval.cpp:155-165): q_hi sized to the genome, then 7, 6, 5
    int q_hi = 2;
    while ((uint64_t{1} << (2 * (q_hi + 1))) <= g->length * 16 && q_hi < 12) ++q_hi;
    std::vector<int> qs{q_hi};
    for (int q : {7, 6, 5})
        if (q < q_hi) qs.push_back(q);
    for (int q : qs) {
        rf->tables.emplace_back();
        if (int rc = build_table(*rf, q, rf->tables.back())) return rc;
    }
    *out = rf.release();
    return SA_OK;
}

void sa_referee_destroy(sa_referee* r) { delete r; }

int sa_referee_align(sa_referee* rf, const sa_params* p, const char* bases, const uint64_t* offsets, uint64_t n_reads,
                     sa_result* results) {
    if (!rf || !p || (n_reads && (!bases || !offsets || !results))) return fail_thread(SA_EINVAL, "null argument");
    if (int rc = sa_validate_params(p)) return rc;
    RF_TRY(cudaSetDevice(rf->device));
    for (uint64_t i = 0; i < n_reads; ++i)
        if (offsets[i + 1] < offsets[i]) return fail_thread(SA_EINVAL, "offsets not ascending");
    const int c = p->confidence_threshold;
    for (uint64_t b0 = 0; b0 < n_reads; b0 += kBatchReads) {
        const uint32_t n = static_cast<uint32_t>(std::min<uint64_t>(kBatchReads, n_reads - b0));
        std::vector<int32_t> dl(n), dmax(n);
        std::vector<uint8_t> fin(n), outcome(n);
        std::vector<uint32_t> todo;
        for (uint32_t i = 0; i < n; ++i) {
            const uint64_t L = offsets[b0 + i + 1] - offsets[b0 + i];
            dmax[i] = effective_dmax(p, L);
            const int full = dmax[i] + c - 1;
            dl[i] = std::min(6, full);  // REF eval.cpp:282
            fin[i] = dl[i] == full;
            sa_result& r = results[b0 + i];
            std::memset(&r, 0, sizeof(r));
            r.kind = SA_NOT_FOUND;
            r.distance = -1;
            if (L >= static_cast<uint64_t>(p->seed_size)) todo.push_back(i);  // REF :277-278
        }
        // stage 1 on the reads that are long enough
        std::vector<uint64_t> so{0};
        std::vector<char> sb;
        std::vector<int32_t> sdl, sdmax;
        std::vector<uint8_t> sfin;
        for (uint32_t i : todo) {
            const uint64_t a = offsets[b0 + i], e = offsets[b0 + i + 1];
            sb.insert(sb.end(), bases + a, bases + e);
            so.push_back(sb.size());
            sdl.push_back(dl[i]);
            sdmax.push_back(dmax[i]);
            sfin.push_back(fin[i]);
        }
        std::vector<sa_result> sres(todo.size());
        std::vector<uint8_t> sout(todo.size());
        if (!todo.empty())
            if (int rc = run_batch(*rf, sb.data(), so.data(), static_cast<uint32_t>(todo.size()), sdl.data(),
                                   sdmax.data(), sfin.data(), c, p->bucket_size, sres.data(), sout.data(), nullptr))
                return rc;
        // stage 2: the full limit for the reads stage 1 could not decide
        std::vector<uint32_t> esc;
        for (size_t k = 0; k < todo.size(); ++k) {
            if (sout[k] == 0) results[b0 + todo[k]] = sres[k];
            else esc.push_back(static_cast<uint32_t>(k));
        }
        if (!esc.empty()) {
            std::vector<uint64_t> eo{0};
            std::vector<char> eb;
            std::vector<int32_t> edl, edm;
            std::vector<uint8_t> efin;
            for (uint32_t k : esc) {
                eb.insert(eb.end(), sb.begin() + static_cast<long>(so[k]), sb.begin() + static_cast<long>(so[k + 1]));
                eo.push_back(eb.size());
                edl.push_back(sdmax[k] + c - 1);
                edm.push_back(sdmax[k]);
                efin.push_back(1);
            }
            std::vector<sa_result> eres(esc.size());
            std::vector<uint8_t> eout(esc.size());
            if (int rc = run_batch(*rf, eb.data(), eo.data(), static_cast<uint32_t>(esc.size()), edl.data(),
                                   edm.data(), efin.data(), c, p->bucket_size, eres.data(), eout.data(), nullptr))
                return rc;
            for (size_t k = 0; k < esc.size(); ++k) results[b0 + todo[esc[k]]] = eres[k];
        }
    }
    return SA_OK;
}

int sa_referee_scan(sa_referee* rf, int32_t d_limit, int32_t bucket_size, const char* bases, const uint64_t* offsets,
                    uint64_t n_reads, uint64_t* hit_offsets, sa_referee_hit* hits, uint64_t cap) {
    if (!rf || !hit_offsets || (n_reads && (!bases || !offsets))) return fail_thread(SA_EINVAL, "null argument");
    if (d_limit < 0) return fail_thread(SA_EINVAL, "d_limit must be non-negative");  // REF edit_distance.cpp:22
    if (bucket_size < 1) return fail_thread(SA_EINVAL, "bucket size must be >= 1");
    RF_TRY(cudaSetDevice(rf->device));
    hit_offsets[0] = 0;
    for (uint64_t b0 = 0; b0 < n_reads; b0 += kBatchReads) {
        const uint32_t n = static_cast<uint32_t>(std::min<uint64_t>(kBatchReads, n_reads - b0));
        std::vector<int32_t> dl(n, d_limit), dmax(n, d_limit);
        std::vector<uint8_t> fin(n, 1), outc(n);
        std::vector<sa_result> res(n);
        std::vector<std::vector<unsigned long long>> h;
        if (int rc = run_batch(*rf, bases, offsets + b0, n, dl.data(), dmax.data(), fin.data(), 1, bucket_size,
                               res.data(), outc.data(), &h))
            return rc;
        for (uint32_t i = 0; i < n; ++i) {
            uint64_t at = hit_offsets[b0 + i];
            for (unsigned long long k : h[i]) {
                if (hits && at < cap) {
                    hits[at].position = (k >> 1) & 0xffffffffull;
                    hits[at].distance = static_cast<int32_t>(k >> 33);
                    hits[at].direction = static_cast<uint8_t>(k & 1);
                    std::memset(hits[at].reserved, 0, sizeof(hits[at].reserved));
                }
                ++at;
            }
            hit_offsets[b0 + i + 1] = at;
        }
    }
    if (hits && hit_offsets[n_reads] > cap) return fail_thread(SA_EINVAL, "hit buffer too small");
    return SA_OK;
}

}  // extern "C"
