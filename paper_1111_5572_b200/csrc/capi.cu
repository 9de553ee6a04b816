// capi.cu -- the C-ABI boundary (include/snap_b200.h) and the host batcher.
//
// One sa_context = one index replica per device (genome planes + seed table
// built on that device) and, per device, a worker that pulls read chunks from
// a shared cursor and streams them through two CUDA streams:
//   H2D bases/offsets -> fast align kernel -> slow (overflow) kernel -> D2H results
// so the copies of chunk k+1 overlap the kernels of chunk k.  Results land in
// input order (chunk i writes results[r0 .. r1)).  No collective is involved:
// replicas are independent (REF include/seedaln/aligner.hpp:112-115 shares the
// index read-only across workers; here across GPUs).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/snap_b200.h"
#include "align_kernels.cuh"
#include "device_index.h"
#include "host_common.h"

using namespace sab;

extern "C" void sab_debug_ktimes(const char* tag);  // align.cu diagnostics (SA_DEBUG_KTIME)

namespace {

thread_local std::string g_thread_err;

}  // namespace

namespace sab {
void set_thread_error(const std::string& msg) { g_thread_err = msg; }
int fail_thread(int code, const std::string& msg) {
    g_thread_err = msg;
    return code;
}
}  // namespace sab

namespace {

#ifndef SA_PIPE_STAGES
#define SA_PIPE_STAGES 6
#endif
constexpr int kPipeStages = SA_PIPE_STAGES;

// Diagnostics (SA_DEBUG_TIMELINE=1): per chunk, events after its H2D (C), seed
// (S), solo (o), resolve (r), warp (w), prune (p), overflow pass (V) and D2H
// (D) kernels on their own streams; printed relative to the batch start.
struct TimelineMark {
    int chunk;
    char tag;
    cudaEvent_t ev;
};
thread_local std::vector<TimelineMark> g_tl;  // per host worker (one per replica)
thread_local int g_tl_chunk = -1;
bool timeline_on() {
    static const bool on = getenv("SA_DEBUG_TIMELINE") != nullptr;
    return on;
}
void tl_mark(char tag, cudaStream_t st) {
    if (!timeline_on()) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    g_tl.push_back({g_tl_chunk, tag, e});
}
void tl_dump(cudaEvent_t base) {
    if (!timeline_on()) return;
    for (auto& m : g_tl) {
        float t = 0;
        cudaEventElapsedTime(&t, base, m.ev);
        fprintf(stderr, "[tl] %d %c %.3f\n", m.chunk, m.tag, t);
        cudaEventDestroy(m.ev);
    }
    g_tl.clear();
}  // chunk buffers in flight per replica (copies run ahead of compute)
constexpr int kCtlWords = 4;  // cursor_fast, cursor_slow, overflow_count, error_flag
// Chunk size of the batch pipeline: about 1/32 of the batch (1/24 until the
// solo kernel got faster: C2 e2e 25.9 ms at 426 k reads per chunk, 25.2 at 328 k), between
// 48 k and 512 k reads.  Each chunk costs a kernel ramp and tail (~15 us), so
// big batches want big chunks (C2, 10 M reads: e2e 152 M reads/s at 48 k,
// 196 M at 512 k), while a 1 M batch wants enough chunks to overlap copy and
// compute (C1: 48 k best).  The 48 k floor scales with the mean read length
// past 128 bases: a long read's kernels cost ~length x d_limit, so a chunk's
// tail (its slowest reads) grows with the length while its copy shrinks in
// relative terms (C3, 500 k x 1 kbp: e2e 167 / 137 / 121 / 112 ms at chunks
// of 48 k / 96 k / 192 k / >= 256 k reads).  SA_CHUNK_READS overrides (tuning).
uint64_t chunk_reads_setting(uint64_t n_reads, uint64_t mean_len) {
    static const long long forced = [] {
        const char* e = getenv("SA_CHUNK_READS");
        return e ? atoll(e) : 0ll;
    }();
    if (forced >= 1024) return static_cast<uint64_t>(forced);
    const uint64_t want = ((n_reads / 32 + 16383) / 16384) * 16384;
    const uint64_t floor = 49152ull * std::max<uint64_t>(1, mean_len / 128);
    return std::min<uint64_t>(512u << 10, std::max<uint64_t>(floor, want));
}
constexpr uint64_t kChunkBytes = 512ull << 20;  // byte cap per chunk (6 stages of device + staging buffers)
#ifndef SA_FAST_CAP
#define SA_FAST_CAP 64    // candidates per read in the shared-memory table (more: the global-table pass)
#endif
#ifndef SA_FAST_HCAP
#define SA_FAST_HCAP 128  // its hash slots (power of two)
#endif
constexpr int kFastCap = SA_FAST_CAP, kFastHcap = SA_FAST_HCAP;
constexpr uint64_t kSlowScratchBudget = 6ull << 30;  // global candidate tables of the overflow kernel

struct Stage {  // one of the two pipeline slots of a replica
    cudaStream_t st = nullptr;
    char* d_bases = nullptr;
    uint64_t bases_cap = 0;
    uint64_t* d_offsets = nullptr;
    sa_result* d_results = nullptr;
    unsigned int* d_overflow = nullptr;
    uint64_t reads_cap = 0;
    unsigned int* d_ctl = nullptr;
    cudaEvent_t k0 = nullptr, km = nullptr, k1 = nullptr;  // fast kernel [k0,km), slow [km,k1)
    cudaEvent_t done = nullptr;                             // after the stage's last D2H
    bool done_pending = false;  // sa_align_device: `done` recorded after the last call's work
    uint4* d_gplanes = nullptr;  // per-warp global read planes of the long-read layouts (AlignLaunch::gplanes)
    uint64_t gplanes_bytes = 0;
    // seed-kernel outputs of the two-kernel path (launch_align_pre)
    uint4* pre_planes = nullptr;
    uint4* pre_recs = nullptr;
    uint2* pre_meta = nullptr;
    unsigned int* pre_list = nullptr;  // solo_kernel's list for the warp kernel; count in the last entry
    unsigned char* pq_pool = nullptr;  // the warp kernel's prune queue (align.cu pq_defer)
    uint64_t pq_cap = 0;
    unsigned int* pq_list = nullptr;
    uint64_t pq_list_cap = 0;
    unsigned long long* pq_ctl = nullptr;  // byte cursor; count | work cursor
    unsigned int* pre_ctl = nullptr;       // kPre read cursors: solo, warp kernel
    uint64_t pre_planes_cap = 0, pre_recs_cap = 0, pre_meta_cap = 0, pre_list_cap = 0;
    // seeded pipeline: input landed / consumed by the seed kernel / aligned /
    // results copied out
    cudaEvent_t e_in = nullptr, e_seeded = nullptr, e_al = nullptr, e_out = nullptr;
    cudaEvent_t e_ov = nullptr;  // the chunk's global-table pass done (seeded pipeline)
    unsigned char* d_gscratch = nullptr;  // that pass's global candidate tables (per stage: passes run concurrently)
    uint64_t gscratch_bytes = 0;
    bool ov_pending = false;     // the stage's last chunk ran a global-table pass
    // packed input (pack.cpp): pinned host planes and their device copy
    uint32_t* h_pack = nullptr;
    uint32_t* d_pack = nullptr;
    uint64_t pack_cap = 0;  // words, all three planes
    // pinned staging for pageable callers: the chunk's bases (+ offsets) in,
    // its results out (copied to the caller once their D2H has landed)
    char* h_in = nullptr;
    uint64_t h_in_cap = 0;
    sa_result* h_res = nullptr;
    uint64_t h_res_cap = 0;
    bool res_pending = false;
    uint64_t res_r0 = 0, res_r1 = 0;
};

int ensure_pack(sa_context* ctx, Stage& s, uint64_t words);

cudaError_t stage_times(Stage& s, float& fast_ms, float& slow_ms) {
    cudaError_t e = cudaEventSynchronize(s.k1);
    if (e != cudaSuccess) return e;
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, s.k0, s.km);
    cudaEventElapsedTime(&b, s.km, s.k1);
    fast_ms += a;
    slow_ms += b;
    return cudaSuccess;
}

struct LaunchShape {
    AlignLaunch proto;  // layout + params fields filled
    int fast_block, fast_grid;
    int pipe_block, pipe_grid;  // the same kernel in the chunked batch pipeline
    int slow_block, slow_grid;
    uint32_t slow_smem_per_warp;
    uint64_t slow_table_bytes;
    uint64_t scratch_bytes;  // global candidate tables of the overflow path
    int slow_cap, slow_hcap;
    uint64_t gplanes_bytes;  // per-warp global read planes (long-read layouts, AlignLaunch::gplanes)
    int stage_slow_grid;     // blocks of a per-chunk global-table pass (seeded pipeline)
};

struct Replica {
    int device = 0;
    int sm_count = 148;
    DeviceIndex ix;
    Stage stage[kPipeStages + 1];  // [0, kPipeStages) batch pipeline, [kPipeStages] sa_align_device
    unsigned long long* d_stats = nullptr;
    unsigned int* d_err = nullptr;         // error flag
    unsigned long long* d_err_read = nullptr;
    // pinned landing zone for the end-of-batch control words: the stats, the
    // error flag and the deferred-read count come back in one synchronisation
    struct HostCtl {
        unsigned long long stats[kNumStats];
        unsigned int err, defer;
    };
    HostCtl* h_ctl = nullptr;
    unsigned char* d_gscratch = nullptr;
    uint64_t gscratch_bytes = 0;
    uint32_t smem_attr = 0;
    cudaEvent_t e_start = nullptr, e_end = nullptr, e_join = nullptr;
    // batch-wide list of reads that overflowed the fast kernel's shared table
    // (absolute read ids), redone by one global-table pass at the end
    unsigned int* d_defer = nullptr;
    unsigned int* d_defer_count = nullptr;
    uint64_t defer_cap = 0;
    // launch layouts already derived for (params, longest read): make_shape
    // queries occupancy and free memory, too slow to repeat per call
    struct ShapeEntry {
        sa_params p;
        uint64_t L;
        LaunchShape sh;
    };
    std::vector<ShapeEntry> shapes;
    // streamed batch path (align_streamed): whole-batch device buffers,
    // per-chunk flags / done counters / byte adjustments, three streams
    struct Streamed {
        char* bases = nullptr;
        uint64_t bases_cap = 0;
        uint64_t* offs = nullptr;
        uint64_t offs_cap = 0;
        sa_result* res = nullptr;
        uint64_t res_cap = 0;
        unsigned int* flags = nullptr;
        unsigned int* done = nullptr;
        long long* adj = nullptr;
        uint64_t chunks_cap = 0;
        unsigned int epoch = 0;
        cudaStream_t ci = nullptr, kk = nullptr, co = nullptr;
        cudaStream_t ov = nullptr;  // seeded pipeline: the chunks' global-table passes, in order (shared scratch)
        cudaEvent_t e_begin = nullptr, e_ready = nullptr, k0 = nullptr, k1 = nullptr, e_end = nullptr;
    } sm;
};


}  // namespace

struct sa_context {
    std::vector<Replica> reps;
    int seed_size = 0;
    uint64_t glen = 0;
    std::string err;
    std::mutex mu;
    float last_e2e_ms = 0, last_kernel_ms = 0, last_slow_ms = 0;
    bool device_timing_pending = false;  // sa_align_device events not yet read
    uint64_t last_launches = 0;
};

namespace {

int fail(sa_context* ctx, int code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    else g_thread_err = msg;
    return code;
}

#define CUDA_TRY(ctx, x)                                                              \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess)                                                        \
            return fail(ctx, SA_ERUNTIME, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

int validate_params(const sa_params* p, std::string& why) {  // REF src/aligner.cpp:11-24
    if (!p) { why = "params is NULL"; return SA_EINVAL; }
    if (p->seed_size < 1 || p->seed_size > 32) { why = "seed-size must be in [1, 32]"; return SA_EINVAL; }
    if (p->seeds_to_try < 1) { why = "seeds-to-try must be >= 1"; return SA_EINVAL; }
    if (p->max_distance < -1) { why = "max-dist must be >= 0 (or -1 for auto)"; return SA_EINVAL; }
    if (p->confidence_threshold < 1) { why = "confidence must be >= 1"; return SA_EINVAL; }
    if (p->max_hits < 1) { why = "max-hits must be >= 1"; return SA_EINVAL; }
    if (p->bucket_size < 1 || p->bucket_size > 64) { why = "bucket-size must be in [1, 64]"; return SA_EINVAL; }
    return SA_OK;
}

inline int round4(int v) { return (v + 3) & ~3; }
inline uint32_t round16(uint64_t v) { return static_cast<uint32_t>((v + 15) & ~15ull); }

// Per-warp shared-memory layout for reads up to Lmax bases.
int make_shape(Replica& rep, const sa_params* p, uint64_t Lmax, LaunchShape& sh, std::string& why) {
    AlignLaunch& a = sh.proto;
    std::memset(&a, 0, sizeof(a));
    a.planes = rep.ix.planes;
    a.glen = rep.ix.glen;
    a.table = rep.ix.table;
    a.n_slots = rep.ix.n_slots;
    a.pool = rep.ix.pool;
    a.s = p->seed_size;
    a.n = p->seeds_to_try;
    a.dmax_param = p->max_distance;
    a.c = p->confidence_threshold;
    a.hmax = p->max_hits;
    a.bs = p->bucket_size;
    a.bs_shift = (a.bs & (a.bs - 1)) == 0 ? __builtin_ctz(static_cast<unsigned>(a.bs)) : -1;
    a.force = p->force_max_dlimit ? 1 : 0;
    if (Lmax < static_cast<uint64_t>(p->seed_size)) Lmax = p->seed_size;
    if (Lmax > (1u << 20)) {
        why = "read longer than 1 Mbp";
        return SA_EINVAL;
    }
    const int L = static_cast<int>(Lmax);
    const int dmax = p->max_distance >= 0 ? p->max_distance : (12 * L + 99) / 100;
    a.dl_max = dmax + p->confidence_threshold - 1;
    a.wbr = (L + 31) / 32 + 2;
    a.wbw = (64 + L + a.dl_max + 31) / 32 + 4;
    a.n_off_cap = round4(std::max(1, std::min(p->seeds_to_try, L - p->seed_size + 1)));
    // per warp: planes {R,C} (two buffers for the read pipeline of reads
    // <= 1 kbp, one otherwise), window, seed records[2][32], probe landing
    // zone[32] + keys[32], offsets[2], LV frontier, read staging, candidate
    // table, stats (align.cu kernel)
    a.prefetch = L <= 1024 ? 1 : 0;
    a.cap = kFastCap;
    a.hcap = kFastHcap;
    if (a.dl_max > 15) {  // long-read layouts: SA_LONG_CAP candidates in the shared table (tuning)
        static const int long_cap = [] {
            const char* e = getenv("SA_LONG_CAP");
            return e ? std::max(16, std::min(1024, atoi(e))) : kFastCap;
        }();
        a.cap = long_cap;
        a.hcap = 1;
        while (a.hcap < 2 * a.cap) a.hcap <<= 1;
    }
    a.lcap = L;  // every read of this layout fits
    a.sbw = a.prefetch ? round4((L + 3) / 4 + 2) : 0;
    auto f_ints_for = [&](int f16) {
        return a.dl_max > 15 ? round4(f16 ? (2 * a.dl_max + 3) : 2 * (2 * a.dl_max + 3)) : 0;
    };
    // gw: the LV reads the genome window from global memory (always for the
    // register LV; for the shared-memory LV only when dropping the staged
    // window fits more warps)
    // gp: the read planes in a per-warp global slot (long reads with the
    // systolic LV, which reads them once per 64 rows; SA_NO_GPLANES keeps them
    // in shared memory).  C4: 10 -> 19 warps per SM.
    static const bool no_gplanes = getenv("SA_NO_GPLANES") != nullptr;
    const bool gp = !no_gplanes && !a.prefetch && SA_LV_LONG && a.dl_max >= SA_BITPAR_MIN_DL && a.dl_max <= kSysMaxDl;
    auto common_for = [&](int f16, int gw) {
        return 16ull * ((gp ? 0 : (a.prefetch ? 4 : 2) * a.wbr) + (gw ? 0 : a.wbw) + 64 + 32) + 8ull * 32 +
               4ull * (2 * a.n_off_cap + f_ints_for(f16)) + 8ull * kNumStats;
    };
    // the pruning batch's area (align.cu prune_batch) closes each warp's share
    // SA_PB_MODE: 0 off, 1 thread-serial wavefront per anchor (default), 2 mask LV (C2 34.6 vs 27.4 ms)
    static const int pb_mode = [] {
        if (getenv("SA_NO_PRUNE_BATCH")) return 0;
        const char* e = getenv("SA_PB_MODE");
        return e ? std::max(0, std::min(2, atoi(e))) : 1;
    }();
    // only where the batch can apply (its bound B <= 5 needs small limits):
    // long-read layouts are shared-memory-limited and keep the space (C3:
    // 138 vs 199 ms per 500 k reads with the area present)
    a.pb_on = a.dl_max <= 15 ? pb_mode : 0;
    // SA_EAGER_PROBES: seeds the seed kernel probes per read (0: all)
    static const int eager = [] {
        const char* e = getenv("SA_EAGER_PROBES");
        return e ? std::max(0, atoi(e)) : 4;
    }();
    a.eager = eager;
    const uint64_t pb_bytes = a.pb_on ? prune_batch_bytes() : 0;
    auto spw_for = [&](int f16, int gw) {
        return round16(common_for(f16, gw) + 8ull * a.sbw + cand_table_bytes(a.cap, a.hcap)) + pb_bytes;
    };
    const uint32_t kMaxSmem = 227 * 1024;
    // warps per block (<= SA_FAST_WARPS) that fit the most warps per SM under
    // shared memory and the 80-register budget (24 warps)
    auto best_block = [&](uint32_t spw, int& warps_sm) {
        int best_w = 0;
        warps_sm = 0;
        for (int w = 1; w <= SA_FAST_WARPS; ++w) {
            if (static_cast<uint64_t>(w) * spw > kMaxSmem) break;
            const int tot = std::min<int>(kRegWarpsPerSM / w, static_cast<int>(kMaxSmem / (w * spw))) * w;
            if (tot >= warps_sm) {
                warps_sm = tot;
                best_w = w;
            }
        }
        return best_w;
    };
    // Layout choice (measured, SA_FORCE_LAYOUT / SA_FORCE_WARPS sweeps):
    // - reads <= 1 kbp (the seeded kernel): the LV reads the genome in place
    //   (C3: 158 -> 149 ms at equal occupancy, 139 ms with the 22 warps/SM the
    //   smaller layout allows) and keeps a 32-bit frontier (16-bit: 219 ms);
    // - longer reads: the 16-bit frontier and the in-place window cost little
    //   per step, so whichever of them fits the most warps per SM wins (C4:
    //   7 warps 372 ms, 8 warps 332-341 ms, both 10 warps 287 ms).
    a.f16 = 0;
    a.gw = 1;
    if (a.dl_max > 15 && !a.prefetch) {
        const bool can16 = L < 32000 && getenv("SA_LV_F16_OFF") == nullptr;
        const int opts[4][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
        int best = -1;
        for (int o = 0; o < 4; ++o) {
            if (opts[o][0] && !can16) continue;
            int wsm = 0;
            best_block(spw_for(opts[o][0], opts[o][1]), wsm);
            if (wsm > best) {
                best = wsm;
                a.f16 = opts[o][0];
                a.gw = opts[o][1];
            }
        }
    }
    if (const char* fl = getenv("SA_FORCE_LAYOUT")) {  // tuning: "f16,gw"
        int f = 0, g = 0;
        if (sscanf(fl, "%d,%d", &f, &g) == 2) {
            a.f16 = f && L < 32000 && a.dl_max > 15;
            a.gw = g || a.dl_max <= 15;
        }
    }
    a.f_ints = f_ints_for(a.f16);
    const uint64_t common = common_for(a.f16, a.gw);
    a.smem_per_warp = spw_for(a.f16, a.gw);
    if (a.smem_per_warp > kMaxSmem) {
        why = "read too long for the shared-memory layout (limit ~60 kbp)";
        return SA_EINVAL;
    }
    int warps_sm = 0;
    int warps = best_block(a.smem_per_warp, warps_sm);
    // shared-memory-limited layouts run best in small blocks (C3: 2-warp
    // blocks 139 ms, 7-warp 149 ms per 500 k reads)
    if (warps_sm < kRegWarpsPerSM && warps > 2 && 2 * a.smem_per_warp <= kMaxSmem) {
        const int tot2 = std::min<int>(kRegWarpsPerSM / 2, static_cast<int>(kMaxSmem / (2 * a.smem_per_warp))) * 2;
        if (tot2 >= warps_sm - 1) warps = 2;
    }
    if (const char* fw = getenv("SA_FORCE_WARPS")) {  // tuning: warps per block
        const int w = atoi(fw);
        if (w >= 1 && w <= SA_FAST_WARPS && static_cast<uint64_t>(w) * a.smem_per_warp <= kMaxSmem) warps = w;
    }
    sh.fast_block = 32 * warps;
    if (getenv("SA_DEBUG_SHAPE"))
        fprintf(stderr, "[shape] L=%d dl_max=%d f16=%d gw=%d smem/warp=%u block=%d warps/SM=%d\n", L, a.dl_max, a.f16,
                a.gw, a.smem_per_warp, warps, warps_sm);
    int bps = 0;
    if (rep.smem_attr < kMaxSmem) {
        if (align_set_smem(kMaxSmem) != cudaSuccess) {
            why = "cudaFuncSetAttribute failed";
            return SA_ERUNTIME;
        }
        rep.smem_attr = kMaxSmem;
    }
    if (align_fast_occupancy(a, sh.fast_block, a.smem_per_warp * warps, &bps) != cudaSuccess || bps < 1) bps = 1;
    sh.fast_grid = bps * rep.sm_count;
    // In the chunked pipeline the kernels of consecutive chunks overlap, and
    // small blocks let the next chunk's blocks take SMs as this one's drain:
    // 2-warp blocks there (C1 e2e 414 -> 419 M reads/s, C2 195 -> 205 M,
    // C3 2.57 -> 2.99 M), the largest block for one big launch (C1 device
    // 506 vs 499 M).  Kept only when 2-warp blocks fit as many warps per SM.
    sh.pipe_block = sh.fast_block;
    sh.pipe_grid = sh.fast_grid;
    {
        int w2 = 0;
        const int pw = getenv("SA_FORCE_WARPS") ? warps : 2;
        if (pw <= warps && static_cast<uint64_t>(pw) * a.smem_per_warp <= kMaxSmem) {
            const int tot = std::min<int>(kRegWarpsPerSM / pw, static_cast<int>(kMaxSmem / (pw * a.smem_per_warp))) * pw;
            best_block(a.smem_per_warp, w2);
            if (tot >= w2 - 1 &&
                align_fast_occupancy(a, 32 * pw, a.smem_per_warp * pw, &bps) == cudaSuccess && bps >= 1) {
                sh.pipe_block = 32 * pw;
                sh.pipe_grid = bps * rep.sm_count;
            }
        }
    }

    // slow path: candidate tables in global memory, worst case n_eff * h_max
    const uint64_t n_eff = static_cast<uint64_t>(std::min(p->seeds_to_try, L - p->seed_size + 1));
    uint64_t cap_slow = std::max<uint64_t>(64, n_eff * static_cast<uint64_t>(p->max_hits));
    if (cap_slow > (1u << 26)) cap_slow = 1u << 26;
    uint64_t hcap_slow = 1;
    while (hcap_slow < 2 * cap_slow) hcap_slow <<= 1;
    sh.slow_cap = static_cast<int>(cap_slow);
    sh.slow_hcap = static_cast<int>(hcap_slow);
    sh.slow_table_bytes = (cand_table_bytes(sh.slow_cap, sh.slow_hcap) + 255) & ~255ull;
    sh.slow_smem_per_warp = round16(common + (gp ? 16ull * 2 * a.wbr : 0)) + pb_bytes;  // planes in shared memory there
    uint64_t slow_warps = std::min<uint64_t>(static_cast<uint64_t>(rep.sm_count) * kRegWarpsPerSM,
                                             std::max<uint64_t>(32, kSlowScratchBudget / sh.slow_table_bytes));
    // 8-warp blocks where shared memory allows: the device path launches this
    // kernel after every batch, usually with nothing to do, and 3552 one-warp
    // blocks cost ~25 us to schedule (C0: 10 k reads in 0.043 ms of kernels)
    const uint64_t sw = std::max<uint64_t>(1, std::min<uint64_t>(8, kMaxSmem / sh.slow_smem_per_warp));
    slow_warps = std::max<uint64_t>(sw, slow_warps / sw * sw);
    sh.slow_block = static_cast<int>(32 * sw);
    sh.slow_grid = static_cast<int>(slow_warps / sw);
    // a chunk's pass has ~0.3% of a chunk's reads: 4 warps per SM are plenty
    sh.stage_slow_grid = static_cast<int>(std::max<uint64_t>(
        1, std::min<uint64_t>(sh.slow_grid, static_cast<uint64_t>(rep.sm_count) * 4 / sw)));
    a.gscratch_per_warp = sh.slow_table_bytes;
    sh.scratch_bytes = slow_warps * sh.slow_table_bytes;
    a.gplanes = nullptr;
    a.gplanes_per_warp = gp ? static_cast<uint32_t>(2 * a.wbr) : 0u;
    sh.gplanes_bytes = gp ? 16ull * a.gplanes_per_warp *
                                static_cast<uint64_t>(std::max(sh.fast_grid * (sh.fast_block / 32),
                                                               sh.pipe_grid * (sh.pipe_block / 32)))
                          : 0;
    // the slow launch overrides cap/hcap/smem_per_warp
    return SA_OK;
}

int cached_shape(Replica& rep, const sa_params* p, uint64_t Lmax, LaunchShape& sh, std::string& why) {
    for (const auto& e : rep.shapes)
        if (e.L == Lmax && std::memcmp(&e.p, p, sizeof(sa_params)) == 0) {
            sh = e.sh;
            return SA_OK;
        }
    if (int rc = make_shape(rep, p, Lmax, sh, why)) return rc;
    if (rep.shapes.size() >= 32) rep.shapes.erase(rep.shapes.begin());
    rep.shapes.push_back({*p, Lmax, sh});
    return SA_OK;
}

int ensure_stage(sa_context* ctx, Stage& s, uint64_t bytes, uint64_t reads) {
    if (!s.st) {
        CUDA_TRY(ctx, cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking));
        CUDA_TRY(ctx, cudaEventCreate(&s.k0));
        CUDA_TRY(ctx, cudaEventCreate(&s.km));
        CUDA_TRY(ctx, cudaEventCreate(&s.k1));
        CUDA_TRY(ctx, cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
        for (cudaEvent_t* e : {&s.e_in, &s.e_seeded, &s.e_al, &s.e_out, &s.e_ov})
            CUDA_TRY(ctx, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        CUDA_TRY(ctx, cudaMalloc(&s.d_ctl, kCtlWords * sizeof(unsigned int)));
    }
    if (bytes > s.bases_cap) {
        if (s.d_bases) cudaFree(s.d_bases);
        s.d_bases = nullptr;
        uint64_t nb = std::max<uint64_t>(bytes, 1 << 16);
        CUDA_TRY(ctx, cudaMalloc(&s.d_bases, nb + 64));
        s.bases_cap = nb;
    }
    if (reads > s.reads_cap) {
        if (s.d_offsets) cudaFree(s.d_offsets);
        if (s.d_results) cudaFree(s.d_results);
        if (s.d_overflow) cudaFree(s.d_overflow);
        s.d_offsets = nullptr;
        s.d_results = nullptr;
        s.d_overflow = nullptr;
        uint64_t nr = std::max<uint64_t>(reads, 1024);
        CUDA_TRY(ctx, cudaMalloc(&s.d_offsets, (nr + 1) * sizeof(uint64_t)));
        CUDA_TRY(ctx, cudaMalloc(&s.d_results, nr * sizeof(sa_result)));
        CUDA_TRY(ctx, cudaMalloc(&s.d_overflow, nr * sizeof(unsigned int)));
        s.reads_cap = nr;
    }
    return SA_OK;
}

int ensure_pack(sa_context* ctx, Stage& s, uint64_t words) {
    if (words <= s.pack_cap) return SA_OK;
    if (s.d_pack) cudaFree(s.d_pack);
    if (s.h_pack) cudaFreeHost(s.h_pack);
    s.d_pack = nullptr;
    s.h_pack = nullptr;
    s.pack_cap = 0;
    const uint64_t w = std::max<uint64_t>(words + words / 4, 1 << 16);
    CUDA_TRY(ctx, cudaMalloc(&s.d_pack, w * sizeof(uint32_t)));
    CUDA_TRY(ctx, cudaHostAlloc(&s.h_pack, w * sizeof(uint32_t), cudaHostAllocDefault));
    s.pack_cap = w;
    return SA_OK;
}

int ensure_host_staging(sa_context* ctx, Stage& s, uint64_t in_bytes, uint64_t reads) {
    if (in_bytes > s.h_in_cap) {
        if (s.h_in) cudaFreeHost(s.h_in);
        s.h_in = nullptr;
        s.h_in_cap = 0;
        const uint64_t b = std::max<uint64_t>(in_bytes + in_bytes / 4, 1 << 20);
        CUDA_TRY(ctx, cudaHostAlloc(&s.h_in, b, cudaHostAllocDefault));
        s.h_in_cap = b;
    }
    if (reads > s.h_res_cap) {
        if (s.h_res) cudaFreeHost(s.h_res);
        s.h_res = nullptr;
        s.h_res_cap = 0;
        const uint64_t r = std::max<uint64_t>(reads + reads / 4, 1 << 12);
        CUDA_TRY(ctx, cudaHostAlloc(&s.h_res, r * sizeof(sa_result), cudaHostAllocDefault));
        s.h_res_cap = r;
    }
    return SA_OK;
}

// True when p is ordinary (pageable) host memory: cudaMemcpyAsync from it
// would be staged synchronously by the driver, so the batcher stages it
// through its own pinned buffers instead.
bool is_pageable(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
}

// the seeded pipeline serves batches whose first chunk holds only reads of
// at most 1 kbp (longer reads later in the batch are deferred)
bool seeded_wanted(const uint64_t* offsets, const std::vector<uint64_t>& bounds) {
    if (bounds.size() < 2) return false;
    for (uint64_t i = bounds[0]; i < bounds[1]; ++i)
        if (offsets[i + 1] < offsets[i] || offsets[i + 1] - offsets[i] > 1024) return false;
    return true;
}

bool use_pre() {
    static const bool v = getenv("SA_NO_PRE") == nullptr;
    return v;
}

// per-read strides of the seed kernel's outputs for a launch layout
int pre_pstride(const AlignLaunch& a) { return 2 * (a.wbr - 1); }  // (nb + 1) blocks per orientation
int pre_rstride(const AlignLaunch& a) { return a.n_off_cap; }

// SA_PRUNE_SPLIT=0 keeps the pruning loop inside the warp kernel
bool prune_split() {
    static const bool on = [] {
        const char* e = getenv("SA_PRUNE_SPLIT");
        return e ? atoi(e) != 0 : true;
    }();
    return on;
}

int ensure_pre(sa_context* ctx, Stage& s, uint64_t n_reads, const LaunchShape& sh) {
    if (!use_pre() || !sh.proto.prefetch) return SA_OK;
    const uint64_t np = n_reads * static_cast<uint64_t>(pre_pstride(sh.proto));
    const uint64_t nr = n_reads * static_cast<uint64_t>(pre_rstride(sh.proto));
    auto grow = [&](auto** p, uint64_t& cap, uint64_t need, size_t elem) -> int {
        if (need <= cap && *p) return SA_OK;
        if (*p) cudaFree(*p);
        *p = nullptr;
        const uint64_t c = std::max<uint64_t>(need, 1024);
        CUDA_TRY(ctx, cudaMalloc(reinterpret_cast<void**>(p), c * elem));
        cap = c;
        return SA_OK;
    };
    if (int rc = grow(&s.pre_planes, s.pre_planes_cap, np, sizeof(uint4))) return rc;
    if (int rc = grow(&s.pre_recs, s.pre_recs_cap, nr, sizeof(uint4))) return rc;
    if (int rc = grow(&s.pre_meta, s.pre_meta_cap, n_reads, sizeof(uint2))) return rc;
    if (int rc = grow(&s.pre_list, s.pre_list_cap, n_reads + 1, sizeof(unsigned int))) return rc;
    if (!s.pre_ctl) CUDA_TRY(ctx, cudaMalloc(&s.pre_ctl, 8 * sizeof(unsigned int)));
    if (prune_split()) {  // ~13% of C2 reads, ~540 B each; a full pool just prunes inline
        uint64_t cap_b = s.pq_cap;
        if (int rc = grow(&s.pq_pool, cap_b, n_reads * 256, 1)) return rc;
        s.pq_cap = cap_b;
        if (int rc = grow(&s.pq_list, s.pq_list_cap, n_reads, sizeof(unsigned int))) return rc;
        if (!s.pq_ctl) CUDA_TRY(ctx, cudaMalloc(&s.pq_ctl, 2 * sizeof(unsigned long long)));
    }
    return SA_OK;
}

void set_pq(AlignLaunch& a, const Stage& s) {
    // the warp kernel's dynamic read cursor (SA_WARP_DYN=0: static striding)
    static const bool warp_dyn = [] {
        const char* e = getenv("SA_WARP_DYN");
        return e ? atoi(e) != 0 : true;
    }();
    if (s.pre_ctl) a.work_cursor = warp_dyn ? s.pre_ctl + 1 : nullptr;
    if (!prune_split() || !s.pq_pool) return;
    a.pq_pool = s.pq_pool;
    a.pq_cap = s.pq_cap;
    a.pq_cursor = s.pq_ctl;
    a.pq_count = reinterpret_cast<unsigned int*>(s.pq_ctl + 1);
    a.pq_cursor2 = a.pq_count + 1;
    a.pq_list = s.pq_list;
}

// a stage's global read-plane slots (kernels of different stages run concurrently)
int ensure_gplanes(sa_context* ctx, Stage& s, const LaunchShape& sh) {
    if (sh.gplanes_bytes > s.gplanes_bytes) {
        if (s.d_gplanes) cudaFree(s.d_gplanes);
        s.d_gplanes = nullptr;
        CUDA_TRY(ctx, cudaMalloc(&s.d_gplanes, sh.gplanes_bytes));
        s.gplanes_bytes = sh.gplanes_bytes;
    }
    return SA_OK;
}

int ensure_scratch(sa_context* ctx, Replica& rep, const LaunchShape& sh) {
    const uint64_t need = sh.scratch_bytes;
    if (need > rep.gscratch_bytes) {
        if (rep.d_gscratch) cudaFree(rep.d_gscratch);
        rep.d_gscratch = nullptr;
        CUDA_TRY(ctx, cudaMalloc(&rep.d_gscratch, need));
        rep.gscratch_bytes = need;
        // hash keys must start empty; tables are self-cleaning afterwards
        CUDA_TRY(ctx, cudaMemset(rep.d_gscratch, 0xff, need));
    }
    return SA_OK;
}

// Device-resident batches are run as slices of this many reads (0: one
// launch sequence for the whole batch).  A slice's seed records and planes
// (288 B per 100 bp read) then stay in L2 between the seed kernel that writes
// them and the kernels that read them, and the next slice overwrites the same
// lines instead of leaving them to be written back.  SA_DEV_CHUNK overrides.
uint64_t dev_chunk_reads() {
    static const uint64_t v = [] {
        const char* e = getenv("SA_DEV_CHUNK");
        return e ? static_cast<uint64_t>(atoll(e)) : uint64_t{0};
    }();
    return v;
}

// Enqueue fast + slow kernels for reads already on the device.
int enqueue_align(sa_context* ctx, Replica& rep, Stage& stg, const LaunchShape& sh,
                  const char* d_bases, const uint64_t* d_offsets, uint64_t base_off,
                  uint64_t n_reads, uint64_t read_base, sa_result* d_results,
                  unsigned long long* d_stats, unsigned int* d_overflow, bool time_it,
                  uint64_t& launches, unsigned int* d_defer_count = nullptr) {
    AlignLaunch a = sh.proto;
    a.bases = d_bases;
    a.offsets = d_offsets;
    a.base_off = base_off;
    a.n_reads = static_cast<uint32_t>(n_reads);
    a.results = d_results;
    a.stats = d_stats;
    a.cursor = stg.d_ctl + 0;
    a.overflow_count = stg.d_ctl + 2;
    a.overflow_list = d_overflow;
    if (d_defer_count) a.overflow_count = d_defer_count;  // batch-wide list, drained at the end
    a.error_flag = rep.d_err;
    a.error_read = rep.d_err_read;
    a.read_base = read_base;
    a.gscratch = rep.d_gscratch;
    if (int rc = ensure_gplanes(ctx, stg, sh)) return rc;
    a.gplanes = a.gplanes_per_warp ? stg.d_gplanes : nullptr;
    CUDA_TRY(ctx, cudaMemsetAsync(stg.d_ctl, 0, kCtlWords * sizeof(unsigned int), stg.st));
    if (time_it) CUDA_TRY(ctx, cudaEventRecord(stg.k0, stg.st));
    if (use_pre() && a.prefetch && stg.pre_planes) {  // seed kernel + align kernel
        a.pre_planes = stg.pre_planes;
        a.pre_recs = stg.pre_recs;
        a.pre_meta = stg.pre_meta;
        a.pre_list = stg.pre_list;
        a.pre_list_count = stg.pre_list + (stg.pre_list_cap - 1);
        set_pq(a, stg);
        a.pre_pstride = pre_pstride(a);
        a.pre_rstride = pre_rstride(a);
        const uint64_t ch = dev_chunk_reads();
        if (ch == 0 || n_reads <= ch) {
            launches += launch_align_pre(a, sh.fast_grid, sh.fast_block, stg.st) - 1;
        } else {  // L2-sized slices reusing one set of seed records (see dev_chunk_reads)
            for (uint64_t r0 = 0; r0 < n_reads; r0 += ch) {
                AlignLaunch c = a;
                c.n_reads = static_cast<uint32_t>(std::min(ch, n_reads - r0));
                c.offsets = d_offsets + r0;
                c.results = d_results + r0;
                c.read_base = read_base + r0;
                launches += launch_align_pre(c, sh.fast_grid, sh.fast_block, stg.st);
            }
            launches -= 1;
        }
    } else {
        launch_align_fast(a, sh.fast_grid, sh.fast_block, stg.st);
    }
    CUDA_TRY(ctx, cudaGetLastError());
    if (time_it) CUDA_TRY(ctx, cudaEventRecord(stg.km, stg.st));
    launches += 1;
    if (d_defer_count) {  // overflowing reads handled by the end-of-batch pass
        if (time_it) CUDA_TRY(ctx, cudaEventRecord(stg.k1, stg.st));
        return SA_OK;
    }
    AlignLaunch b = a;
    b.pq_pool = nullptr;  // the global-table kernel prunes inline
    b.cursor = stg.d_ctl + 1;
    b.work_list = d_overflow;
    b.work_count = stg.d_ctl + 2;
    b.overflow_list = nullptr;
    b.overflow_count = nullptr;
    b.cap = sh.slow_cap;
    b.hcap = sh.slow_hcap;
    b.smem_per_warp = sh.slow_smem_per_warp;
    b.sbw = 0;
    b.prefetch = 0;
    launch_align_slow(b, sh.slow_grid, sh.slow_block, stg.st);
    CUDA_TRY(ctx, cudaGetLastError());
    if (time_it) CUDA_TRY(ctx, cudaEventRecord(stg.k1, stg.st));
    launches += 1;
    return SA_OK;
}

int check_errors(sa_context* ctx, Replica& rep) {
    unsigned int flag = 0;
    unsigned long long first = 0;
    CUDA_TRY(ctx, cudaMemcpy(&flag, rep.d_err, sizeof(flag), cudaMemcpyDeviceToHost));
    if (flag & 2u) {
        CUDA_TRY(ctx, cudaMemset(rep.d_err, 0, sizeof(unsigned int)));
        return fail(ctx, SA_ERUNTIME, "candidate table overflow on the global-table path "
                                      "(seeds_to_try * max_hits above 2^26)");
    }
    if (flag) {
        CUDA_TRY(ctx, cudaMemcpy(&first, rep.d_err_read, sizeof(first), cudaMemcpyDeviceToHost));
        CUDA_TRY(ctx, cudaMemset(rep.d_err, 0, sizeof(unsigned int)));
        CUDA_TRY(ctx, cudaMemset(rep.d_err_read, 0xff, sizeof(unsigned long long)));
        return fail(ctx, SA_EINVAL, "reverse_complement: non-base character (read " +
                                        std::to_string(first) +
                                        " holds a character outside {A,C,G,T,N})");
    }
    return SA_OK;
}

int ensure_defer(sa_context* ctx, Replica& rep, uint64_t n) {
    if (!rep.d_defer_count) CUDA_TRY(ctx, cudaMalloc(&rep.d_defer_count, sizeof(unsigned int)));
    if (n > rep.defer_cap) {
        if (rep.d_defer) cudaFree(rep.d_defer);
        rep.d_defer = nullptr;
        const uint64_t c = std::max<uint64_t>(n, 1 << 16);
        CUDA_TRY(ctx, cudaMalloc(&rep.d_defer, c * sizeof(unsigned int)));
        rep.defer_cap = c;
    }
    return SA_OK;
}

// End-of-batch overflow pass: the reads whose candidates overflowed the fast
// kernel's shared table (their ids collected batch-wide, nothing committed for
// them) are gathered on the host, copied once, aligned by the global-table
// kernel and scattered into results.  Keeping this out of the chunk pipeline
// means no kernel ever queues behind the persistent fast kernel of the next
// chunk.  Returns the number of reads redone.
int cached_shape(Replica& rep, const sa_params* p, uint64_t Lmax, LaunchShape& sh, std::string& why);
int ensure_scratch(sa_context* ctx, Replica& rep, const LaunchShape& sh);

int overflow_pass(sa_context* ctx, Replica& rep, Stage& stg, const sa_params* params, const char* bases,
                  const uint64_t* offsets, sa_result* results, uint64_t& launches, uint64_t& n_done) {
    unsigned int n = 0;
    n_done = 0;
    CUDA_TRY(ctx, cudaMemcpyAsync(&n, rep.d_defer_count, sizeof(n), cudaMemcpyDeviceToHost, stg.st));
    CUDA_TRY(ctx, cudaStreamSynchronize(stg.st));
    if (n == 0) return SA_OK;
    std::vector<unsigned int> ids(n);
    CUDA_TRY(ctx, cudaMemcpy(ids.data(), rep.d_defer, n * sizeof(unsigned int), cudaMemcpyDeviceToHost));
    std::vector<uint64_t> offs(n + 1, 0);
    uint64_t Lmax = 0;
    for (unsigned i = 0; i < n; ++i) {
        const uint64_t L = offsets[ids[i] + 1] - offsets[ids[i]];
        offs[i + 1] = offs[i] + L;
        Lmax = std::max(Lmax, L);
    }
    // deferred reads: table overflows and (streaming) reads longer than the
    // fast launch's layout -- the global-table kernel gets its own layout
    LaunchShape sh;
    {
        std::string why;
        if (int rc = cached_shape(rep, params, Lmax, sh, why)) return fail(ctx, rc, why);
        if (int rc = ensure_scratch(ctx, rep, sh)) return rc;
    }
    std::vector<char> buf(offs[n]);
    for (unsigned i = 0; i < n; ++i)
        std::memcpy(buf.data() + offs[i], bases + offsets[ids[i]], offs[i + 1] - offs[i]);
    if (int rc = ensure_stage(ctx, stg, offs[n], n)) return rc;
    CUDA_TRY(ctx, cudaMemcpyAsync(stg.d_bases, buf.data(), offs[n], cudaMemcpyHostToDevice, stg.st));
    CUDA_TRY(ctx, cudaMemcpyAsync(stg.d_offsets, offs.data(), (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice,
                                  stg.st));
    CUDA_TRY(ctx, cudaMemsetAsync(stg.d_ctl, 0, kCtlWords * sizeof(unsigned int), stg.st));
    AlignLaunch b = sh.proto;
    b.bases = stg.d_bases;
    b.offsets = stg.d_offsets;
    b.base_off = 0;
    b.n_reads = n;
    b.results = stg.d_results;
    b.stats = rep.d_stats;
    b.cursor = stg.d_ctl + 1;
    b.work_list = nullptr;  // every read of this launch
    b.work_count = rep.d_defer_count;  // == n
    b.overflow_list = nullptr;
    b.overflow_count = nullptr;
    b.error_flag = rep.d_err;
    b.error_read = rep.d_err_read;
    b.read_base = 0;
    b.gscratch = rep.d_gscratch;
    b.gplanes = nullptr;
    b.cap = sh.slow_cap;
    b.hcap = sh.slow_hcap;
    b.smem_per_warp = sh.slow_smem_per_warp;
    b.sbw = 0;
    b.prefetch = 0;
    launch_align_slow(b, sh.slow_grid, sh.slow_block, stg.st);
    CUDA_TRY(ctx, cudaGetLastError());
    ++launches;
    std::vector<sa_result> out(n);
    CUDA_TRY(ctx, cudaMemcpyAsync(out.data(), stg.d_results, n * sizeof(sa_result), cudaMemcpyDeviceToHost, stg.st));
    CUDA_TRY(ctx, cudaStreamSynchronize(stg.st));
    for (unsigned i = 0; i < n; ++i) results[ids[i]] = out[i];
    n_done = n;
    return SA_OK;
}

void add_stats(sa_stats* dst, const unsigned long long* src) {
    uint64_t* d = reinterpret_cast<uint64_t*>(dst);
    for (int i = 0; i < kNumStats; ++i) d[i] += src[i];
}


// ---------------------------------------------------------------- streamed batch path
// cuStreamWriteValue32 / cuStreamWaitValue32 (stream memory operations,
// executed by the front end, no SM) through the runtime's driver entry
// points: chunk flags for the kernel and done-count gates for the D2H.
typedef int (*StreamValueFn)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
struct MemOps {
    StreamValueFn write = nullptr, wait = nullptr;
    bool ok = false;
};
const MemOps& memops() {
    static MemOps m = [] {
        MemOps r;
        cudaDriverEntryPointQueryResult q1, q2;
        void* w = nullptr;
        void* v = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1) == cudaSuccess &&
            cudaGetDriverEntryPoint("cuStreamWaitValue32", &v, cudaEnableDefault, &q2) == cudaSuccess &&
            q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && w && v) {
            r.write = reinterpret_cast<StreamValueFn>(w);
            r.wait = reinterpret_cast<StreamValueFn>(v);
            r.ok = true;
        }
        cudaGetLastError();
        return r;
    }();
    return m;
}
constexpr unsigned kWaitGeq = 0x0;  // CU_STREAM_WAIT_VALUE_GEQ
constexpr int kStreamShift = 14;    // 16 k reads per chunk

// Opt-in (SA_STREAM=1): one launch per batch with the in-kernel read
// preparation, chunk flags via stream memory ops.  The default batch path is
// the seeded chunk pipeline (seed kernel + align kernel per chunk), which
// measured faster on C1 once the seed kernel existed.
bool streaming_wanted(const Replica& rep, uint64_t n_reads, const uint64_t* offsets, const void* results) {
    if (!getenv("SA_STREAM") || getenv("SA_OVERFLOW_KERNEL")) return false;
    (void)results;
    if (n_reads < (2ull << kStreamShift) || !memops().ok) return false;
    (void)rep;
    uint64_t L = 0;  // the first chunk decides the layout; longer reads are deferred
    const uint64_t m = std::min<uint64_t>(n_reads, 1ull << kStreamShift);
    for (uint64_t i = 0; i < m; ++i) {
        if (offsets[i + 1] < offsets[i]) return false;
        L = std::max(L, offsets[i + 1] - offsets[i]);
    }
    return L <= 1024;
}

template <typename T>
int grow(sa_context* ctx, T** p, uint64_t& cap, uint64_t need) {
    if (need <= cap && *p) return SA_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    const uint64_t c = std::max<uint64_t>(need, 1024);
    CUDA_TRY(ctx, cudaMalloc(p, c * sizeof(T)));
    cap = c;
    return SA_OK;
}

// One launch for the whole batch: chunks of 16 k reads are copied in on one
// stream, each followed by a flag write; the persistent kernel (another
// stream) waits per chunk for its flag, and a third stream waits on each
// chunk's done count before copying its results out.  No kernel boundary per
// chunk, no tail per chunk.
int align_streamed(sa_context* ctx, Replica& rep, const sa_params* params, const char* bases,
                   const uint64_t* offsets, uint64_t n_reads, sa_result* results, sa_stats* out_stats,
                   float& e2e_ms, float& k_ms, uint64_t& launches) {
    auto& S = rep.sm;
    const MemOps& mo = memops();
    CUDA_TRY(ctx, cudaSetDevice(rep.device));
    if (!S.ci) {
        CUDA_TRY(ctx, cudaStreamCreateWithFlags(&S.ci, cudaStreamNonBlocking));
        CUDA_TRY(ctx, cudaStreamCreateWithFlags(&S.kk, cudaStreamNonBlocking));
        CUDA_TRY(ctx, cudaStreamCreateWithFlags(&S.co, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&S.e_begin, &S.e_ready, &S.k0, &S.k1, &S.e_end}) CUDA_TRY(ctx, cudaEventCreate(e));
    }
    const uint64_t CH = 1ull << kStreamShift;  // first chunk
    static const int sh0 = getenv("SA_STREAM_SHIFT0") ? atoi(getenv("SA_STREAM_SHIFT0")) : 14;
    static const int sh1 = getenv("SA_STREAM_SHIFT") ? atoi(getenv("SA_STREAM_SHIFT")) : 16;
    const uint64_t n_chunks = stream_chunk_of(static_cast<uint32_t>(n_reads - 1), sh0, sh1) + 1;
    auto cbeg = [&](uint64_t c) -> uint64_t {
        return std::min<uint64_t>(n_reads, stream_chunk_begin(static_cast<uint32_t>(c), sh0, sh1));
    };
    // layout: the first chunk's longest read, rounded up to 32 bases
    uint64_t L0 = 0;
    for (uint64_t i = 0; i < std::min(n_reads, CH); ++i) L0 = std::max(L0, offsets[i + 1] - offsets[i]);
    L0 = std::max<uint64_t>((L0 + 31) & ~31ull, 32);
    LaunchShape sh;
    {
        std::string why;
        if (int rc = cached_shape(rep, params, L0, sh, why)) return fail(ctx, rc, why);
        if (int rc = ensure_scratch(ctx, rep, sh)) return rc;
    }
    // chunk byte placement: each chunk's bytes start on a 128-byte boundary,
    // so no cache line holds two chunks (the kernel reads bytes through L1)
    std::vector<long long> adj(n_chunks);
    std::vector<uint64_t> dpos(n_chunks + 1, 0);
    bool bad_bounds = false;
    for (uint64_t c = 0; c < n_chunks; ++c) {
        const uint64_t r0 = cbeg(c), r1 = cbeg(c + 1);
        uint64_t bytes = 0;
        if (offsets[r1] >= offsets[r0]) bytes = offsets[r1] - offsets[r0];
        else bad_bounds = true;
        adj[c] = static_cast<long long>(dpos[c]) - static_cast<long long>(offsets[r0]);
        dpos[c + 1] = (dpos[c] + bytes + 127) & ~127ull;
    }
    if (bad_bounds) return fail(ctx, SA_EINVAL, "offsets not ascending");
    {
        if (int rc = grow(ctx, &S.bases, S.bases_cap, dpos[n_chunks] + 64)) return rc;
        if (int rc = grow(ctx, &S.offs, S.offs_cap, n_reads + 1)) return rc;
        if (int rc = grow(ctx, &S.res, S.res_cap, n_reads)) return rc;
        if (S.chunks_cap < n_chunks || !S.flags) {
            uint64_t c1 = S.chunks_cap, c2 = S.chunks_cap, c3 = S.chunks_cap;
            if (int rc = grow(ctx, &S.flags, c1, n_chunks)) return rc;
            if (int rc = grow(ctx, &S.done, c2, n_chunks)) return rc;
            if (int rc = grow(ctx, &S.adj, c3, n_chunks)) return rc;
            CUDA_TRY(ctx, cudaMemset(S.flags, 0, c1 * sizeof(unsigned int)));
            S.chunks_cap = std::min(c1, std::min(c2, c3));
            S.epoch = 0;
        }
    }
    if (int rc = ensure_defer(ctx, rep, n_reads)) return rc;
    if (int rc = ensure_stage(ctx, rep.stage[0], 0, 0)) return rc;  // the overflow pass runs there
    const unsigned epoch = ++S.epoch == 0 ? ++S.epoch : S.epoch;
    // Per-chunk copy-out needs pinned results: a D2H into pageable memory
    // blocks the host until it runs, and chunk c finishes only once later
    // chunks have been flagged (the kernel prefetches two reads ahead).
    cudaPointerAttributes pa{};
    const bool gated = cudaPointerGetAttributes(&pa, results) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();

    // ---- setup on the copy-in stream, then the kernel
    CUDA_TRY(ctx, cudaEventRecord(S.e_begin, S.ci));
    CUDA_TRY(ctx, cudaMemsetAsync(S.done, 0, n_chunks * sizeof(unsigned int), S.ci));
    CUDA_TRY(ctx, cudaMemsetAsync(rep.d_defer_count, 0, sizeof(unsigned int), S.ci));
    CUDA_TRY(ctx, cudaMemsetAsync(rep.d_stats, 0, kNumStats * sizeof(unsigned long long), S.ci));
    CUDA_TRY(ctx, cudaMemcpyAsync(S.adj, adj.data(), n_chunks * sizeof(long long), cudaMemcpyHostToDevice, S.ci));
    CUDA_TRY(ctx, cudaEventRecord(S.e_ready, S.ci));
    CUDA_TRY(ctx, cudaStreamWaitEvent(S.kk, S.e_ready, 0));
    CUDA_TRY(ctx, cudaStreamWaitEvent(S.co, S.e_ready, 0));
    AlignLaunch a = sh.proto;
    a.bases = S.bases;
    a.offsets = S.offs;
    a.base_off = 0;
    a.n_reads = static_cast<uint32_t>(n_reads);
    a.results = S.res;
    a.stats = rep.d_stats;
    a.cursor = rep.stage[0].d_ctl;  // unused by the pipelined kernel
    a.overflow_list = rep.d_defer;
    a.overflow_count = rep.d_defer_count;
    a.error_flag = rep.d_err;
    a.error_read = rep.d_err_read;
    a.read_base = 0;
    a.gscratch = rep.d_gscratch;
    if (int rc = ensure_gplanes(ctx, rep.stage[0], sh)) return rc;
    a.gplanes = a.gplanes_per_warp ? rep.stage[0].d_gplanes : nullptr;
    a.chunk_flag = S.flags;
    a.chunk_done = S.done;
    a.chunk_adj = S.adj;
    a.epoch = epoch;
    a.chunk_shift0 = sh0;
    a.chunk_shift = sh1;
    const bool precopy = getenv("SA_STREAM_PRECOPY") != nullptr;  // diagnostics: all copies before the kernel
    auto launch = [&]() -> int {
        CUDA_TRY(ctx, cudaEventRecord(S.k0, S.kk));
        launch_align_fast(a, sh.fast_grid, sh.fast_block, S.kk);
        CUDA_TRY(ctx, cudaGetLastError());
        CUDA_TRY(ctx, cudaEventRecord(S.k1, S.kk));
        ++launches;
        return SA_OK;
    };
    if (!precopy)
        if (int rc = launch()) return rc;

    // ---- chunks: validate, copy in, flag; gate and copy out
    int bad = SA_OK;
    std::vector<uint64_t> zero_offs;
    for (uint64_t c = 0; c < n_chunks; ++c) {
        const uint64_t r0 = cbeg(c), r1 = cbeg(c + 1);
        const uint64_t* src_offs = offsets + r0;
        for (uint64_t i = r0; i < r1; ++i)
            if (offsets[i + 1] < offsets[i]) {
                if (!bad) bad = fail(ctx, SA_EINVAL, "offsets not ascending");
                break;
            }
        if (bad) {  // keep the kernel safe: zero-length reads at the chunk start
            zero_offs.assign(r1 - r0 + 1, offsets[r0]);
            src_offs = zero_offs.data();
        } else {
            CUDA_TRY(ctx, cudaMemcpyAsync(S.bases + dpos[c], bases + offsets[r0], offsets[r1] - offsets[r0],
                                          cudaMemcpyHostToDevice, S.ci));
        }
        CUDA_TRY(ctx, cudaMemcpyAsync(S.offs + r0, src_offs, (r1 - r0 + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice,
                                      S.ci));
        if (bad) CUDA_TRY(ctx, cudaStreamSynchronize(S.ci));  // zero_offs is reused
        if (mo.write(S.ci, reinterpret_cast<unsigned long long>(S.flags + c), epoch, 0) != 0)
            return fail(ctx, SA_ERUNTIME, "cuStreamWriteValue32 failed");
        if (gated) {
            if (mo.wait(S.co, reinterpret_cast<unsigned long long>(S.done + c), static_cast<unsigned>(r1 - r0),
                        kWaitGeq) != 0)
                return fail(ctx, SA_ERUNTIME, "cuStreamWaitValue32 failed");
            CUDA_TRY(ctx, cudaMemcpyAsync(results + r0, S.res + r0, (r1 - r0) * sizeof(sa_result),
                                          cudaMemcpyDeviceToHost, S.co));
        }
    }
    if (precopy) {
        CUDA_TRY(ctx, cudaStreamSynchronize(S.ci));
        if (int rc = launch()) return rc;
    }
    CUDA_TRY(ctx, cudaStreamWaitEvent(S.co, S.k1, 0));  // stats are final once the kernel ends
    if (!gated)
        CUDA_TRY(ctx, cudaMemcpyAsync(results, S.res, n_reads * sizeof(sa_result), cudaMemcpyDeviceToHost, S.co));
    CUDA_TRY(ctx, cudaEventRecord(S.e_end, S.co));
    CUDA_TRY(ctx, cudaEventSynchronize(S.e_end));
    cudaEventElapsedTime(&e2e_ms, S.e_begin, S.e_end);
    cudaEventElapsedTime(&k_ms, S.k0, S.k1);
    if (bad) return bad;
    {
        unsigned int flag = 0;
        CUDA_TRY(ctx, cudaMemcpy(&flag, rep.d_err, sizeof(flag), cudaMemcpyDeviceToHost));
        if (flag & 4u) {
            CUDA_TRY(ctx, cudaMemset(rep.d_err, 0, sizeof(unsigned int)));
            return fail(ctx, SA_ERUNTIME, "streamed batch: a chunk never arrived (timeout)");
        }
    }
    uint64_t redone = 0;
    if (int rc = overflow_pass(ctx, rep, rep.stage[0], params, bases, offsets, results, launches, redone)) return rc;
    if (redone) {  // the pass ran after e_end: extend the measured span
        CUDA_TRY(ctx, cudaEventRecord(S.e_end, rep.stage[0].st));
        CUDA_TRY(ctx, cudaEventSynchronize(S.e_end));
        cudaEventElapsedTime(&e2e_ms, S.e_begin, S.e_end);
    }
    unsigned long long h[kNumStats];
    CUDA_TRY(ctx, cudaMemcpy(h, rep.d_stats, sizeof(h), cudaMemcpyDeviceToHost));
    std::memset(out_stats, 0, sizeof(sa_stats));
    add_stats(out_stats, h);
    return check_errors(ctx, rep);
}


// ---------------------------------------------------------------- seeded chunk pipeline
// Batch path for reads <= 1 kbp: three streams per replica.
//   copy-in:  H2D of chunk k into stage k % S (after seed(k - S) consumed it)
//   compute:  align(k - 1), then seed(k) -- one kernel at a time, so the seed
//             kernel never waits for SMs held by a persistent align kernel
//   copy-out: D2H of chunk k's results once align(k) is done
// Reads longer than the layout are deferred (status 3) to the overflow pass.
struct SeededChunk {
    uint64_t r0 = 0, r1 = 0;
    int k = 0;  // chunk number (diagnostics)
    int stage = 0;
    bool ov = false;  // its overflowing reads get their own global-table pass
    cudaStream_t cs = nullptr;  // compute stream
    AlignLaunch a{};
    int grid = 0, block = 0;
};

int seeded_pipeline(sa_context* ctx, Replica& rep, const sa_params* params, const char* bases,
                    const uint64_t* offsets, const std::vector<uint64_t>& bounds, std::atomic<size_t>& next,
                    uint64_t n_reads, sa_result* results, float& e2e_ms, float& k_ms, uint64_t& launches,
                    sa_stats* out) {
    const auto t_host0 = std::chrono::steady_clock::now();  // diagnostics (SA_DEBUG_PIPE)
    auto& S = rep.sm;
    if (!S.ci) {
        CUDA_TRY(ctx, cudaStreamCreateWithFlags(&S.ci, cudaStreamNonBlocking));
        CUDA_TRY(ctx, cudaStreamCreateWithFlags(&S.kk, cudaStreamNonBlocking));
        CUDA_TRY(ctx, cudaStreamCreateWithFlags(&S.co, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&S.e_begin, &S.e_ready, &S.k0, &S.k1, &S.e_end}) CUDA_TRY(ctx, cudaEventCreate(e));
    }
    if (!S.ov) CUDA_TRY(ctx, cudaStreamCreateWithFlags(&S.ov, cudaStreamNonBlocking));
    for (int j = 0; j < kPipeStages; ++j) rep.stage[j].ov_pending = false;
    // Reads that overflow the shared candidate table are redone chunk by
    // chunk by the global-table kernel on its own stream, between the
    // chunk's align kernels and its copy-out (SA_CHUNK_OVERFLOW=0: one pass at
    // the end of the batch, which measured ~3.5 ms of a 29 ms C2 call).
    static const bool chunk_overflow = [] {
        const char* e = getenv("SA_CHUNK_OVERFLOW");
        return e ? atoi(e) != 0 : true;
    }();
    const size_t n_chunks = bounds.size() - 1;
    LaunchShape sh;
    uint64_t shape_L = 0;
    int k = 0, bad = SA_OK;
    SeededChunk pend;
    bool have_pend = false;
    const bool packed = pack_enabled(is_pageable(bases));
    // pageable caller buffers go through pinned staging (SA_NO_STAGING: hand
    // them to cudaMemcpyAsync as they are, which the driver stages synchronously)
    static const bool no_staging = getenv("SA_NO_STAGING") != nullptr;
    const bool stage_in = !packed && !no_staging && is_pageable(bases);
    const bool stage_out = !no_staging && is_pageable(results);
    // a stage's pinned results, once their D2H has landed, go to the caller
    for (int j = 0; j < kPipeStages; ++j) rep.stage[j].res_pending = false;  // nothing owed from a failed call
    auto drain_results = [&](Stage& st) -> int {
        if (!st.res_pending) return SA_OK;
        CUDA_TRY(ctx, cudaEventSynchronize(st.e_out));
        parallel_copy(results + st.res_r0, st.h_res, (st.res_r1 - st.res_r0) * sizeof(sa_result));
        st.res_pending = false;
        return SA_OK;
    };
    // Chunk k's seed and align kernels run on its stage's own stream, so the
    // kernels of consecutive chunks share the GPU: the next chunk's blocks
    // fill the SMs a kernel's tail leaves idle (C1 e2e 367 -> 405 M reads/s).
    // SA_PIPE_SINGLE=1 keeps one compute stream (align(k-1), then seed(k)).
    const bool multi = getenv("SA_PIPE_SINGLE") == nullptr;
    const bool dbg_span = getenv("SA_DEBUG_PIPE") != nullptr;
    const bool dbg = dbg_span && !multi;  // per-kernel trail: single compute stream only
    std::vector<std::pair<char, cudaEvent_t>> trail;  // diagnostics: compute-stream marks
    auto mark = [&](char what) {
        if (!dbg) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, S.kk);
        trail.emplace_back(what, e);
    };
    auto align_pending = [&]() -> int {
        Stage& st = rep.stage[pend.stage];
        CUDA_TRY(ctx, cudaStreamWaitEvent(pend.cs, st.e_out, 0));  // results buffer free (no-op first time)
        mark('w');
        g_tl_chunk = static_cast<int>(pend.k);
        if (timeline_on()) sab::g_timeline_hook = tl_mark;
        launches += launch_align_seeded(pend.a, pend.grid, pend.block, pend.cs) - 1;
        sab::g_timeline_hook = nullptr;
        mark('a');
        CUDA_TRY(ctx, cudaGetLastError());
        ++launches;
        CUDA_TRY(ctx, cudaEventRecord(st.e_al, pend.cs));
        if (pend.ov) {  // the chunk's overflowing reads: global-table kernel on the chunk's stream
            // with the stage's own tables, so the passes of different chunks run
            // concurrently (one shared stream serialised them: each waited for the
            // previous chunk's slowest overflowing read)
            const uint64_t need = static_cast<uint64_t>(sh.stage_slow_grid) * (sh.slow_block / 32) *
                                  sh.slow_table_bytes;
            if (need > st.gscratch_bytes) {
                if (st.d_gscratch) cudaFree(st.d_gscratch);
                st.d_gscratch = nullptr;
                st.gscratch_bytes = 0;
                CUDA_TRY(ctx, cudaMalloc(&st.d_gscratch, need));
                CUDA_TRY(ctx, cudaMemset(st.d_gscratch, 0xff, need));  // hash keys start empty (self-cleaning after)
                st.gscratch_bytes = need;
            }
            AlignLaunch b = pend.a;
            b.gscratch = st.d_gscratch;
            b.cursor = st.d_ctl + 1;
            b.work_list = st.d_overflow;
            b.work_count = st.d_ctl + 2;
            b.overflow_list = nullptr;
            b.overflow_count = nullptr;
            b.cap = sh.slow_cap;
            b.hcap = sh.slow_hcap;
            b.smem_per_warp = sh.slow_smem_per_warp;
            b.sbw = 0;
            b.prefetch = 0;
            b.pq_pool = nullptr;
            b.pre_list = nullptr;
            b.pre_list_count = nullptr;
            launch_align_slow(b, sh.stage_slow_grid, sh.slow_block, pend.cs);
            CUDA_TRY(ctx, cudaGetLastError());
            ++launches;
            CUDA_TRY(ctx, cudaEventRecord(st.e_ov, pend.cs));
            tl_mark('V', pend.cs);
            CUDA_TRY(ctx, cudaStreamWaitEvent(S.co, st.e_ov, 0));
        } else {
            CUDA_TRY(ctx, cudaStreamWaitEvent(S.co, st.e_al, 0));
        }
        if (stage_out) {
            if (int rc = drain_results(st)) return rc;  // this stage's previous chunk
            CUDA_TRY(ctx, cudaMemcpyAsync(st.h_res, st.d_results, (pend.r1 - pend.r0) * sizeof(sa_result),
                                          cudaMemcpyDeviceToHost, S.co));
            st.res_pending = true;
            st.res_r0 = pend.r0;
            st.res_r1 = pend.r1;
        } else {
            CUDA_TRY(ctx, cudaMemcpyAsync(results + pend.r0, st.d_results, (pend.r1 - pend.r0) * sizeof(sa_result),
                                          cudaMemcpyDeviceToHost, S.co));
        }
        CUDA_TRY(ctx, cudaEventRecord(st.e_out, S.co));
        tl_mark('D', S.co);
        return SA_OK;
    };
    for (;;) {
        const size_t c = next.fetch_add(1);
        if (c >= n_chunks) break;
        const uint64_t r0 = bounds[c], r1 = bounds[c + 1];
        uint64_t Lc = 0, Lmin = ~0ull;
        bool desc = false;
        for (uint64_t i = r0; i < r1; ++i) {  // branch-free scan
            const uint64_t o0 = offsets[i], o1 = offsets[i + 1];
            desc |= o1 < o0;
            const uint64_t li = o1 - o0;
            Lc = li > Lc ? li : Lc;
            Lmin = li < Lmin ? li : Lmin;
        }
        if (desc) {
            bad = fail(ctx, SA_EINVAL, "offsets not ascending");
            break;
        }
        // one length for the whole chunk: the offsets need not be copied
        const uint32_t fixed = (Lmin == Lc && Lc > 0 && Lc < (1u << 30)) ? static_cast<uint32_t>(Lc) : 0u;
        // a chunk whose reads all fit the layout redoes its overflows itself;
        // longer reads (deferred by the seed kernel) go to the end-of-batch pass
        // (host-packed chunks keep no ASCII copy; reads > 256 bases: one pass at the end
        // of the batch -- C3's per-chunk passes cost 112 vs 101 ms of e2e in their tails)
        const bool ov = chunk_overflow && !packed && Lc <= 256;
        Lc = std::min<uint64_t>(Lc, 1024);
        if (k == 0 || Lc > shape_L) {
            std::string w;
            if ((bad = cached_shape(rep, params, std::max(Lc, shape_L), sh, w))) {
                fail(ctx, bad, w);
                break;
            }
            shape_L = std::max(Lc, shape_L);
            if ((bad = ensure_scratch(ctx, rep, sh))) break;
        }
        const int si = k % kPipeStages;
        Stage& st = rep.stage[si];
        const uint64_t b0 = offsets[r0], b1 = offsets[r1];
        if ((bad = ensure_stage(ctx, st, b1 - b0, r1 - r0))) break;
        if ((bad = ensure_pre(ctx, st, r1 - r0, sh))) break;
        if (stage_in || stage_out) {
            // the stage's pinned buffers may grow (the chunk ramp): first
            // finish with their previous chunk (its H2D landed, its results
            // handed to the caller)
            if (k >= kPipeStages) {
                if ((bad = drain_results(st))) break;
                CUDA_TRY(ctx, cudaEventSynchronize(st.e_in));
            }
            if ((bad = ensure_host_staging(ctx, st, stage_in ? (b1 - b0) + (r1 - r0 + 1) * sizeof(uint64_t) + 8 : 0,
                                           stage_out ? r1 - r0 : 0)))
                break;
        }
        if (k == 0) {
            if ((bad = ensure_defer(ctx, rep, n_reads))) break;
            CUDA_TRY(ctx, cudaEventRecord(S.e_begin, S.ci));
            CUDA_TRY(ctx, cudaMemsetAsync(rep.d_defer_count, 0, sizeof(unsigned int), S.ci));
            CUDA_TRY(ctx, cudaMemsetAsync(rep.d_stats, 0, kNumStats * sizeof(unsigned long long), S.ci));
            CUDA_TRY(ctx, cudaEventRecord(S.e_ready, S.ci));
            CUDA_TRY(ctx, cudaStreamWaitEvent(S.kk, S.e_ready, 0));
            CUDA_TRY(ctx, cudaStreamWaitEvent(S.co, S.e_ready, 0));
        }
        // align(k - 1) first: its data is ready, and the host packs chunk k next
        if (have_pend) {
            if (int rc = align_pending()) return rc;
            have_pend = false;
        }
        // copy in (the stage's bytes are free once seed(k - S) has run)
        const uint64_t wpp = packed ? pack_words_per_plane(b1 - b0) : 0;
        if (packed) {
            if ((bad = ensure_pack(ctx, st, 3 * wpp))) break;
            // the stage's host planes are free once their last copy landed
            if (k >= kPipeStages) CUDA_TRY(ctx, cudaEventSynchronize(st.e_in));
            pack_planar(bases + b0, b1 - b0, st.h_pack, wpp);
        }
        const char* src_b = bases + b0;
        const uint64_t* src_o = offsets + r0;
        if (stage_in) {
            // the host copies chunk k into the stage's pinned buffer (free once
            // its previous H2D landed) while the GPU runs the earlier chunks
            if (k >= kPipeStages) CUDA_TRY(ctx, cudaEventSynchronize(st.e_in));
            const uint64_t ob = ((b1 - b0) + 7) & ~7ull;
            parallel_copy(st.h_in, bases + b0, b1 - b0);
            src_b = st.h_in;
            if (!fixed) {
                std::memcpy(st.h_in + ob, offsets + r0, (r1 - r0 + 1) * sizeof(uint64_t));
                src_o = reinterpret_cast<const uint64_t*>(st.h_in + ob);
            }
        }
        if (k >= kPipeStages) CUDA_TRY(ctx, cudaStreamWaitEvent(S.ci, st.e_seeded, 0));
        if (st.ov_pending) CUDA_TRY(ctx, cudaStreamWaitEvent(S.ci, st.e_ov, 0));  // its pass reads the bytes too
        st.ov_pending = ov;
        static const bool no_copy = getenv("SA_DEBUG_NOCOPY") != nullptr;  // diagnostics: compute-only pipeline
        if (no_copy) {  // the batch's bytes from a device-resident copy instead of the H2D (timing only)
            static char* d_all = nullptr;
            static uint64_t all_cap = 0;
            const uint64_t tot = offsets[n_reads] - offsets[0];
            if (tot > all_cap) {
                if (d_all) cudaFree(d_all);
                CUDA_TRY(ctx, cudaMalloc(&d_all, tot));
                CUDA_TRY(ctx, cudaMemcpy(d_all, bases + offsets[0], tot, cudaMemcpyHostToDevice));
                all_cap = tot;
            }
            CUDA_TRY(ctx, cudaMemcpyAsync(st.d_bases, d_all + (b0 - offsets[0]), b1 - b0, cudaMemcpyDeviceToDevice, S.ci));
        } else if (packed)
            CUDA_TRY(ctx, cudaMemcpyAsync(st.d_pack, st.h_pack, 3 * wpp * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                          S.ci));
        else
            CUDA_TRY(ctx, cudaMemcpyAsync(st.d_bases, src_b, b1 - b0, cudaMemcpyHostToDevice, S.ci));
        if (!fixed)
            CUDA_TRY(ctx, cudaMemcpyAsync(st.d_offsets, src_o, (r1 - r0 + 1) * sizeof(uint64_t),
                                          cudaMemcpyHostToDevice, S.ci));
        CUDA_TRY(ctx, cudaEventRecord(st.e_in, S.ci));
        g_tl_chunk = k;
        tl_mark('C', S.ci);
        // compute: seed(k), then align(k - 1)
        AlignLaunch a = sh.proto;
        a.bases = st.d_bases;
        a.offsets = st.d_offsets;
        a.base_off = b0;
        a.n_reads = static_cast<uint32_t>(r1 - r0);
        a.results = st.d_results;
        a.stats = rep.d_stats;
        a.cursor = st.d_ctl;
        a.overflow_list = ov ? st.d_overflow : rep.d_defer;
        a.overflow_count = ov ? st.d_ctl + 2 : rep.d_defer_count;
        a.error_flag = rep.d_err;
        a.error_read = rep.d_err_read;
        a.read_base = r0;
        a.gscratch = rep.d_gscratch;
        a.gplanes = nullptr;  // seeded layouts (reads <= 1 kbp) keep their planes in shared memory
        a.pre_planes = st.pre_planes;
        a.pre_recs = st.pre_recs;
        a.pre_meta = st.pre_meta;
        a.pre_list = st.pre_list;
        a.pre_list_count = st.pre_list + (st.pre_list_cap - 1);
        set_pq(a, st);
        a.pre_pstride = pre_pstride(a);
        a.pre_rstride = pre_rstride(a);
        a.packed = packed ? st.d_pack : nullptr;
        a.pk_wpp = wpp;
        a.fixed_len = fixed;
        cudaStream_t cs = multi ? st.st : S.kk;
        CUDA_TRY(ctx, cudaStreamWaitEvent(cs, st.e_in, 0));
        if (k == 0) CUDA_TRY(ctx, cudaEventRecord(S.k0, cs));
        if (ov) CUDA_TRY(ctx, cudaMemsetAsync(st.d_ctl, 0, kCtlWords * sizeof(unsigned int), cs));
        mark('W');
        launch_seed(a, cs);
        mark('s');
        tl_mark('S', cs);
        CUDA_TRY(ctx, cudaGetLastError());
        ++launches;
        CUDA_TRY(ctx, cudaEventRecord(st.e_seeded, cs));
        pend.r0 = r0;
        pend.r1 = r1;
        pend.k = k;
        pend.stage = si;
        pend.cs = cs;
        pend.a = a;
        pend.grid = sh.pipe_grid;
        pend.block = sh.pipe_block;
        pend.ov = ov;
        have_pend = true;
        if (multi) {
            if (int rc = align_pending()) return rc;
            have_pend = false;
        }
        ++k;
    }
    if (have_pend && !bad)
        if (int rc = align_pending()) return rc;
    if (multi)  // join the stage streams into the compute stream
        for (int j = 0; j < kPipeStages && j < k; ++j) {
            CUDA_TRY(ctx, cudaEventRecord(rep.stage[j].done, rep.stage[j].st));
            CUDA_TRY(ctx, cudaStreamWaitEvent(S.kk, rep.stage[j].done, 0));
        }
    if (k > 0) {  // and the global-table passes
        CUDA_TRY(ctx, cudaEventRecord(rep.stage[0].e_ov, S.ov));
        CUDA_TRY(ctx, cudaStreamWaitEvent(S.kk, rep.stage[0].e_ov, 0));
    }
    if (k > 0) {
        CUDA_TRY(ctx, cudaEventRecord(S.k1, S.kk));
        CUDA_TRY(ctx, cudaStreamWaitEvent(S.co, S.k1, 0));
        if (!rep.h_ctl) CUDA_TRY(ctx, cudaHostAlloc(&rep.h_ctl, sizeof(Replica::HostCtl), cudaHostAllocDefault));
        CUDA_TRY(ctx, cudaMemcpyAsync(rep.h_ctl->stats, rep.d_stats, sizeof(rep.h_ctl->stats), cudaMemcpyDeviceToHost,
                                      S.co));
        CUDA_TRY(ctx, cudaMemcpyAsync(&rep.h_ctl->err, rep.d_err, sizeof(unsigned int), cudaMemcpyDeviceToHost, S.co));
        CUDA_TRY(ctx, cudaMemcpyAsync(&rep.h_ctl->defer, rep.d_defer_count, sizeof(unsigned int),
                                      cudaMemcpyDeviceToHost, S.co));
        CUDA_TRY(ctx, cudaEventRecord(S.e_end, S.co));
    }
    if (dbg_span && k > 0) CUDA_TRY(ctx, cudaEventRecord(S.e_ready, S.ci));  // copy-in span end (diagnostics)
    const auto t_enq = std::chrono::steady_clock::now();
    CUDA_TRY(ctx, cudaStreamSynchronize(S.co));
    CUDA_TRY(ctx, cudaStreamSynchronize(S.ci));
    for (int j = 0; j < kPipeStages; ++j)
        if (int rc = drain_results(rep.stage[j])) return rc;
    if (k > 0) tl_dump(S.e_begin);
    if (dbg_span && k > 0) {
        float ci = 0, kb = 0, ke = 0;
        cudaEventElapsedTime(&ci, S.e_begin, S.e_ready);
        cudaEventElapsedTime(&kb, S.e_begin, S.k0);
        cudaEventElapsedTime(&ke, S.e_begin, S.k1);
        const double host_ms = std::chrono::duration<double, std::milli>(t_enq - t_host0).count();
        const double all_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count();
        fprintf(stderr, "[pipe] chunks=%d copy-in ends %.3f ms, compute %.3f..%.3f ms; host enqueue %.3f ms, host total %.3f ms\n",
                k, ci, kb, ke, host_ms, all_ms);
        // kernel time vs waiting: 'W'/'w' marks precede seed/align, 's'/'a' follow
        float seed = 0, al = 0, wait = 0;
        for (size_t i = 1; i < trail.size(); ++i) {
            float d = 0;
            cudaEventElapsedTime(&d, trail[i - 1].second, trail[i].second);
            if (trail[i].first == 's') seed += d;
            else if (trail[i].first == 'a') al += d;
            else wait += d;
        }
        fprintf(stderr, "[pipe] seed %.3f ms, align %.3f ms, between kernels %.3f ms\n", seed, al, wait);
        sab_debug_ktimes("pipe");
    }
    for (auto& t : trail) cudaEventDestroy(t.second);
    std::memset(out, 0, sizeof(sa_stats));
    if (bad || k == 0) return bad;
    cudaEventElapsedTime(&k_ms, S.k0, S.k1);
    if (rep.h_ctl->defer == 0 && rep.h_ctl->err == 0) {  // the common case: one synchronisation in all
        cudaEventElapsedTime(&e2e_ms, S.e_begin, S.e_end);
        add_stats(out, rep.h_ctl->stats);
        return SA_OK;
    }
    // the overflow pass (stage 0's stream) follows everything above
    if (int rc = ensure_stage(ctx, rep.stage[0], 0, 0)) return rc;
    uint64_t redone = 0;
    if (int rc = overflow_pass(ctx, rep, rep.stage[0], params, bases, offsets, results, launches, redone)) return rc;
    CUDA_TRY(ctx, cudaEventRecord(S.e_end, rep.stage[0].st));
    CUDA_TRY(ctx, cudaEventSynchronize(S.e_end));
    cudaEventElapsedTime(&e2e_ms, S.e_begin, S.e_end);
    unsigned long long h[kNumStats];
    CUDA_TRY(ctx, cudaMemcpy(h, rep.d_stats, sizeof(h), cudaMemcpyDeviceToHost));
    add_stats(out, h);
    return check_errors(ctx, rep);
}

}  // namespace

extern "C" {

void sa_default_params(sa_params* out) {  // REF include/seedaln/aligner.hpp:20-26
    out->seed_size = 20;
    out->seeds_to_try = 25;
    out->max_distance = -1;
    out->confidence_threshold = 2;
    out->max_hits = 300;
    out->bucket_size = 32;
    out->force_max_dlimit = 0;
}

int sa_validate_params(const sa_params* p) {
    std::string why;
    int rc = validate_params(p, why);
    if (rc) g_thread_err = why;
    return rc;
}

int sa_seed_offsets(uint64_t read_length, int32_t s, int32_t n, int32_t* out, int32_t* count) {
    // REF src/aligner.cpp:50-79 (host copy of the kernel's compute_offsets)
    *count = 0;
    if (s < 1 || n < 1 || read_length < static_cast<uint64_t>(s)) return SA_OK;
    if (s > 32) {
        g_thread_err = "seed size must be in [1, 32]";
        return SA_EINVAL;
    }
    const int64_t max_off = static_cast<int64_t>(read_length) - s;
    int cnt = 0;
    uint64_t used = 0;
    auto emit = [&](int shift) {
        if ((used >> shift) & 1ull) return;
        used |= 1ull << shift;
        for (int64_t o = shift; o <= max_off && cnt < n; o += s) out[cnt++] = static_cast<int32_t>(o);
    };
    emit(0);
    for (int level = 1; (int64_t{1} << level) <= 4 * int64_t{s} && cnt < n; ++level)
        for (int64_t odd = 1; odd < (int64_t{1} << level) && cnt < n; odd += 2)
            emit(static_cast<int>((odd * s) >> level));
    *count = cnt;
    return SA_OK;
}

const char* sa_last_error(const sa_context* ctx) {
    return ctx ? ctx->err.c_str() : g_thread_err.c_str();
}

int sa_create(const uint64_t* packed_words, uint64_t n_packed, const uint64_t* nmask_words,
              uint64_t n_nmask, uint64_t genome_length, int32_t seed_size, const int32_t* devices,
              int32_t n_devices, sa_context** out) {
    if (!out) return fail(nullptr, SA_EINVAL, "out is NULL");
    *out = nullptr;
    if (seed_size < 1 || seed_size > 32)  // REF src/seed_index.cpp:81-82
        return fail(nullptr, SA_EINVAL, "seed size must be in [1, 32]");
    if (genome_length < static_cast<uint64_t>(seed_size))  // REF :83-84
        return fail(nullptr, SA_EINVAL, "genome shorter than seed size");
    if (genome_length > 0xffffffffull - 64)
        return fail(nullptr, SA_EINVAL, "genome longer than 2^32 - 64 bases");
    if (n_packed != (genome_length + 31) / 32 || n_nmask != (genome_length + 63) / 64)
        return fail(nullptr, SA_EFORMAT, "packed/n-mask word counts do not match genome length");
    std::vector<int> devs;
    if (!devices || n_devices <= 0) devs.push_back(0);
    else devs.assign(devices, devices + n_devices);
    int have = 0;
    if (cudaGetDeviceCount(&have) != cudaSuccess || have == 0)
        return fail(nullptr, SA_ERUNTIME, "no CUDA device visible");
    auto* ctx = new sa_context;
    ctx->seed_size = seed_size;
    ctx->glen = genome_length;
    ctx->reps.resize(devs.size());
    std::vector<std::string> errs(devs.size());
    std::vector<int> codes(devs.size(), 0);
    auto build = [&](size_t i) {
        Replica& rep = ctx->reps[i];
        rep.device = devs[i];
        if (cudaSetDevice(rep.device) != cudaSuccess) {
            codes[i] = SA_ERUNTIME;
            errs[i] = "cudaSetDevice failed";
            return;
        }
        cudaDeviceGetAttribute(&rep.sm_count, cudaDevAttrMultiProcessorCount, rep.device);
        if (const char* e = getenv("SA_L2_FETCH")) {  // tuning: L2 fetch granularity hint (bytes)
            cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, static_cast<size_t>(atoi(e)));
        }
        cudaStream_t st;
        cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        std::string e;
        if (build_device_index(packed_words, n_packed, nmask_words, n_nmask, genome_length,
                               seed_size, st, &rep.ix, e) != 0) {
            codes[i] = SA_ERUNTIME;
            errs[i] = "index build on device " + std::to_string(rep.device) + ": " + e;
        }
        cudaStreamDestroy(st);
        if (!codes[i]) {
            if (cudaMalloc(&rep.d_stats, kNumStats * sizeof(unsigned long long)) != cudaSuccess ||
                cudaMalloc(&rep.d_err, sizeof(unsigned int)) != cudaSuccess ||
                cudaMemset(rep.d_err, 0, sizeof(unsigned int)) != cudaSuccess ||
                cudaMalloc(&rep.d_err_read, sizeof(unsigned long long)) != cudaSuccess ||
                cudaMemset(rep.d_err_read, 0xff, sizeof(unsigned long long)) != cudaSuccess ||
                cudaEventCreate(&rep.e_start) != cudaSuccess ||
                cudaEventCreate(&rep.e_end) != cudaSuccess ||
                cudaEventCreate(&rep.e_join) != cudaSuccess) {
                codes[i] = SA_ERUNTIME;
                errs[i] = "device allocation failed";
            }
        }
    };
    if (devs.size() == 1) {
        build(0);
    } else {
        std::vector<std::thread> th;
        for (size_t i = 0; i < devs.size(); ++i) th.emplace_back(build, i);
        for (auto& t : th) t.join();
    }
    for (size_t i = 0; i < devs.size(); ++i) {
        if (codes[i]) {
            int c = codes[i];
            std::string m = errs[i];
            sa_destroy(ctx);
            return fail(nullptr, c, m);
        }
    }
    *out = ctx;
    return SA_OK;
}

void sa_destroy(sa_context* ctx) {
    if (!ctx) return;
    for (auto& rep : ctx->reps) {
        cudaSetDevice(rep.device);
        for (auto& s : rep.stage) {
            if (s.st) cudaStreamSynchronize(s.st);
            if (s.d_bases) cudaFree(s.d_bases);
            if (s.d_offsets) cudaFree(s.d_offsets);
            if (s.d_results) cudaFree(s.d_results);
            if (s.d_overflow) cudaFree(s.d_overflow);
            if (s.d_ctl) cudaFree(s.d_ctl);
            if (s.k0) cudaEventDestroy(s.k0);
            if (s.km) cudaEventDestroy(s.km);
            if (s.k1) cudaEventDestroy(s.k1);
            if (s.done) cudaEventDestroy(s.done);
            for (cudaEvent_t e : {s.e_in, s.e_seeded, s.e_al, s.e_out})
                if (e) cudaEventDestroy(e);
            if (s.pre_planes) cudaFree(s.pre_planes);
            if (s.pre_recs) cudaFree(s.pre_recs);
            if (s.pre_meta) cudaFree(s.pre_meta);
            if (s.pre_list) cudaFree(s.pre_list);
            if (s.pq_pool) cudaFree(s.pq_pool);
            if (s.pq_list) cudaFree(s.pq_list);
            if (s.pq_ctl) cudaFree(s.pq_ctl);
            if (s.pre_ctl) cudaFree(s.pre_ctl);
            if (s.d_pack) cudaFree(s.d_pack);
            if (s.h_pack) cudaFreeHost(s.h_pack);
            if (s.h_in) cudaFreeHost(s.h_in);
            if (s.h_res) cudaFreeHost(s.h_res);
            if (s.st) cudaStreamDestroy(s.st);
        }
        if (rep.d_stats) cudaFree(rep.d_stats);
        if (rep.d_err) cudaFree(rep.d_err);
        if (rep.d_err_read) cudaFree(rep.d_err_read);
        if (rep.h_ctl) cudaFreeHost(rep.h_ctl);
        if (rep.d_gscratch) cudaFree(rep.d_gscratch);
        for (auto& sg : rep.stage) {
            if (sg.d_gplanes) cudaFree(sg.d_gplanes);
            if (sg.d_gscratch) cudaFree(sg.d_gscratch);
        }
        if (rep.d_defer) cudaFree(rep.d_defer);
        for (void* q : {static_cast<void*>(rep.sm.bases), static_cast<void*>(rep.sm.offs),
                        static_cast<void*>(rep.sm.res), static_cast<void*>(rep.sm.flags),
                        static_cast<void*>(rep.sm.done), static_cast<void*>(rep.sm.adj)})
            if (q) cudaFree(q);
        for (cudaStream_t q : {rep.sm.ci, rep.sm.kk, rep.sm.co, rep.sm.ov})
            if (q) cudaStreamDestroy(q);
        for (cudaEvent_t e : {rep.sm.e_begin, rep.sm.e_ready, rep.sm.k0, rep.sm.k1, rep.sm.e_end})
            if (e) cudaEventDestroy(e);
        if (rep.d_defer_count) cudaFree(rep.d_defer_count);
        if (rep.e_start) cudaEventDestroy(rep.e_start);
        if (rep.e_end) cudaEventDestroy(rep.e_end);
        if (rep.e_join) cudaEventDestroy(rep.e_join);
        free_device_index(&rep.ix);
    }
    delete ctx;
}

int sa_index_info(const sa_context* ctx, uint64_t* distinct_seeds, uint64_t* total_positions,
                  uint64_t* device_bytes) {
    if (!ctx || ctx->reps.empty()) return fail(nullptr, SA_EINVAL, "null context");
    const DeviceIndex& ix = ctx->reps[0].ix;
    if (distinct_seeds) *distinct_seeds = ix.n_distinct;
    if (total_positions) *total_positions = ix.n_positions;
    if (device_bytes) *device_bytes = ix.device_bytes;
    return SA_OK;
}

int sa_index_seed_size(const sa_context* ctx, int32_t* seed_size) {
    if (!ctx || !seed_size) return fail(nullptr, SA_EINVAL, "null argument");
    *seed_size = ctx->seed_size;
    return SA_OK;
}

int sa_align_batch(sa_context* ctx, const sa_params* params, const char* bases,
                   const uint64_t* offsets, uint64_t n_reads, sa_result* results, sa_stats* stats) {
    if (!ctx) return fail(nullptr, SA_EINVAL, "null context");
    std::lock_guard<std::mutex> lock(ctx->mu);
    std::string why;
    if (int rc = validate_params(params, why)) return fail(ctx, rc, why);
    if (params->seed_size != ctx->seed_size)  // REF src/aligner.cpp:119-121
        return fail(ctx, SA_EINVAL, "index seed size does not match params");
    if (n_reads == 0) {
        ctx->last_e2e_ms = ctx->last_kernel_ms = 0;
        ctx->last_launches = 0;
        return SA_OK;
    }
    if (!bases || !offsets || !results) return fail(ctx, SA_EINVAL, "null buffer");
    if (n_reads >= 0xffffffffull) return fail(ctx, SA_EINVAL, "too many reads in one batch");
    if (ctx->reps.size() == 1 && streaming_wanted(ctx->reps[0], n_reads, offsets, results)) {
        float e2e = 0, kms = 0;
        uint64_t launches = 0;
        sa_stats st;
        const int rc = align_streamed(ctx, ctx->reps[0], params, bases, offsets, n_reads, results, &st, e2e, kms,
                                      launches);
        if (rc) return rc;
        ctx->last_e2e_ms = e2e;
        ctx->last_kernel_ms = kms;
        ctx->last_slow_ms = 0;
        ctx->device_timing_pending = false;
        ctx->last_launches = launches;
        if (stats) {
            uint64_t* d = reinterpret_cast<uint64_t*>(stats);
            const uint64_t* v = reinterpret_cast<const uint64_t*>(&st);
            for (size_t i = 0; i < sizeof(sa_stats) / 8; ++i) d[i] += v[i];
        }
        return SA_OK;
    }
    // chunk boundaries (reads and bytes bounded).  Offsets are validated per
    // chunk inside the pipeline, so the host scan overlaps the GPU's work on
    // the previous chunk; a bad chunk stops the batch before it is enqueued.
    // Chunk sizes ramp up (16 k, 32 k, ... reads) so the first kernel starts
    // after a short copy; the GPU is busy with chunk k while chunk k+1 copies.
    const uint64_t chunk_reads = chunk_reads_setting(n_reads, (offsets[n_reads] - offsets[0]) / n_reads);
    std::vector<uint64_t> bounds{0};
    {
        // sizes ramp up (16 k, 32 k, ...) so the first kernel starts after a
        // short copy, and back down at the end so little compute is left once
        // the last copy lands; equal chunks in between
        std::vector<uint64_t> up;
        static const uint64_t ramp0 = [] {  // SA_RAMP0: first ramp size (tuning; >= chunk size: no ramp)
            const char* e = getenv("SA_RAMP0");
            return e ? static_cast<uint64_t>(atoll(e)) : uint64_t{1} << 14;
        }();
        for (uint64_t s = std::min<uint64_t>(chunk_reads, std::max<uint64_t>(ramp0, 1024)); s < chunk_reads; s *= 2)
            up.push_back(s);
        uint64_t ramp = 0;
        for (uint64_t s : up) ramp += 2 * s;
        std::vector<uint64_t> sizes;
        if (n_reads >= ramp + chunk_reads) {
            sizes = up;
            const uint64_t mid = n_reads - ramp, m = (mid + chunk_reads - 1) / chunk_reads;
            for (uint64_t i = 0; i < m; ++i) sizes.push_back(mid / m + (i < mid % m ? 1 : 0));
            sizes.insert(sizes.end(), up.rbegin(), up.rend());
        } else {
            uint64_t left = n_reads, s = up.empty() ? chunk_reads : up[0];
            while (left) {
                sizes.push_back(std::min(left, s));
                left -= sizes.back();
                s = std::min(chunk_reads, 2 * s);
            }
        }
        for (uint64_t s : sizes) {
            const uint64_t b = bounds.back();
            uint64_t e = b + s;
            while (e > b + 1 && offsets[e] - offsets[b] > kChunkBytes) e = b + (e - b) / 2;
            bounds.push_back(e);
            while (bounds.back() < b + s) {  // byte-capped: finish this size in pieces
                const uint64_t bb = bounds.back();
                uint64_t ee = b + s;
                while (ee > bb + 1 && offsets[ee] - offsets[bb] > kChunkBytes) ee = bb + (ee - bb) / 2;
                bounds.push_back(ee);
            }
        }
    }
    const size_t n_chunks = bounds.size() - 1;
    std::atomic<size_t> next{0};
    std::vector<int> codes(ctx->reps.size(), 0);
    std::vector<std::string> msgs(ctx->reps.size());
    std::vector<sa_stats> part(ctx->reps.size());
    std::vector<float> e2e(ctx->reps.size(), 0), kms(ctx->reps.size(), 0), kslow(ctx->reps.size(), 0);
    std::vector<uint64_t> launches(ctx->reps.size(), 0);

    auto worker = [&](size_t ri) {
        Replica& rep = ctx->reps[ri];
        sa_context local_err;  // per-worker error sink
        auto run = [&]() -> int {
            if (cudaSetDevice(rep.device) != cudaSuccess) return fail(&local_err, SA_ERUNTIME, "cudaSetDevice");
            LaunchShape sh;
            uint64_t shape_L = 0;
            int k = 0, bad = SA_OK;
            // SA_OVERFLOW_KERNEL (test hook): overflow kernel after every chunk
            const bool defer = getenv("SA_OVERFLOW_KERNEL") == nullptr;
            if (defer && use_pre() && seeded_wanted(offsets, bounds)) {
                uint64_t lnch = 0;
                const int rc = seeded_pipeline(&local_err, rep, params, bases, offsets, bounds, next, n_reads, results,
                                               e2e[ri], kms[ri], lnch, &part[ri]);
                launches[ri] += lnch;
                return rc;
            }
            static const bool no_staging = getenv("SA_NO_STAGING") != nullptr;
            const bool stage_in = !no_staging && is_pageable(bases);
            for (;;) {
                size_t c = next.fetch_add(1);
                if (c >= n_chunks) break;
                const uint64_t r0 = bounds[c], r1 = bounds[c + 1];
                uint64_t Lc = 0;
                for (uint64_t i = r0; i < r1; ++i) {
                    if (offsets[i + 1] < offsets[i]) {
                        bad = fail(&local_err, SA_EINVAL, "offsets not ascending");
                        break;
                    }
                    Lc = std::max(Lc, offsets[i + 1] - offsets[i]);
                }
                if (bad) break;
                if (k == 0 || Lc > shape_L) {  // launch layout for the longest read so far
                    std::string w;
                    if ((bad = cached_shape(rep, params, std::max(Lc, shape_L), sh, w))) {
                        fail(&local_err, bad, w);
                        break;
                    }
                    shape_L = std::max(Lc, shape_L);
                    if ((bad = ensure_scratch(&local_err, rep, sh))) break;
                }
                const uint64_t b0 = offsets[r0], b1 = offsets[r1];
                Stage& stg = rep.stage[k % kPipeStages];
                if ((bad = ensure_stage(&local_err, stg, b1 - b0, r1 - r0))) break;
                if (k < kPipeStages) {
                    if (k == 0) {
                        if (defer && (bad = ensure_defer(&local_err, rep, n_reads))) break;
                        if (defer)
                            CUDA_TRY(&local_err, cudaMemsetAsync(rep.d_defer_count, 0, sizeof(unsigned int),
                                                                 rep.stage[0].st));
                        CUDA_TRY(&local_err, cudaMemsetAsync(rep.d_stats, 0, kNumStats * sizeof(unsigned long long),
                                                             rep.stage[0].st));
                        CUDA_TRY(&local_err, cudaEventRecord(rep.e_start, rep.stage[0].st));
                    } else {
                        CUDA_TRY(&local_err, cudaStreamWaitEvent(stg.st, rep.e_start, 0));
                    }
                }
                // stage reuse: collect the kernel events of its previous chunk
                if (k >= kPipeStages) CUDA_TRY(&local_err, stage_times(stg, kms[ri], kslow[ri]));
                // pageable callers: the chunk goes through the stage's pinned buffer
                // (free: the stage's previous chunk has finished, stage_times above),
                // copied by the host pool while the GPU works on the other stages
                // (C4 from numpy buffers: 128 -> ~80 ms per 50 k reads)
                const char* src_b = bases + b0;
                const uint64_t* src_o = offsets + r0;
                if (stage_in) {
                    const uint64_t ob = ((b1 - b0) + 7) & ~7ull;
                    if ((bad = ensure_host_staging(&local_err, stg, ob + (r1 - r0 + 1) * sizeof(uint64_t), 0))) break;
                    parallel_copy(stg.h_in, bases + b0, b1 - b0);
                    std::memcpy(stg.h_in + ob, offsets + r0, (r1 - r0 + 1) * sizeof(uint64_t));
                    src_b = stg.h_in;
                    src_o = reinterpret_cast<const uint64_t*>(stg.h_in + ob);
                }
                CUDA_TRY(&local_err, cudaMemcpyAsync(stg.d_bases, src_b, b1 - b0, cudaMemcpyHostToDevice, stg.st));
                CUDA_TRY(&local_err, cudaMemcpyAsync(stg.d_offsets, src_o, (r1 - r0 + 1) * sizeof(uint64_t),
                                                     cudaMemcpyHostToDevice, stg.st));
                if ((bad = ensure_pre(&local_err, stg, r1 - r0, sh))) break;
                if (int rc = enqueue_align(&local_err, rep, stg, sh, stg.d_bases, stg.d_offsets, b0, r1 - r0, r0,
                                           stg.d_results, rep.d_stats, defer ? rep.d_defer : stg.d_overflow, true,
                                           launches[ri], defer ? rep.d_defer_count : nullptr))
                    return rc;
                CUDA_TRY(&local_err, cudaMemcpyAsync(results + r0, stg.d_results, (r1 - r0) * sizeof(sa_result),
                                                     cudaMemcpyDeviceToHost, stg.st));
                ++k;
            }
            if (bad || k == 0) {  // drain whatever was enqueued before returning
                for (int j = 0; j < kPipeStages; ++j)
                    if (rep.stage[j].st) cudaStreamSynchronize(rep.stage[j].st);
                std::memset(&part[ri], 0, sizeof(sa_stats));
                return bad;
            }
            for (int j = 0; j < kPipeStages && j < k; ++j)
                CUDA_TRY(&local_err, stage_times(rep.stage[(k - 1 - j) % kPipeStages], kms[ri], kslow[ri]));
            for (int j = 1; j < kPipeStages && j < k; ++j) {  // join the other stages into stage[0]
                CUDA_TRY(&local_err, cudaEventRecord(rep.stage[j].done, rep.stage[j].st));
                CUDA_TRY(&local_err, cudaStreamWaitEvent(rep.stage[0].st, rep.stage[j].done, 0));
            }
            if (defer) {
                uint64_t redone = 0;
                if (int rc = overflow_pass(&local_err, rep, rep.stage[0], params, bases, offsets, results,
                                           launches[ri], redone))
                    return rc;
            }
            CUDA_TRY(&local_err, cudaEventRecord(rep.e_end, rep.stage[0].st));
            CUDA_TRY(&local_err, cudaEventSynchronize(rep.e_end));
            cudaEventElapsedTime(&e2e[ri], rep.e_start, rep.e_end);
            unsigned long long h[kNumStats];
            CUDA_TRY(&local_err, cudaMemcpy(h, rep.d_stats, sizeof(h), cudaMemcpyDeviceToHost));
            std::memset(&part[ri], 0, sizeof(sa_stats));
            add_stats(&part[ri], h);
            return check_errors(&local_err, rep);
        };
        codes[ri] = run();
        if (codes[ri]) msgs[ri] = local_err.err;
    };
    if (ctx->reps.size() == 1) {
        worker(0);
    } else {
        std::vector<std::thread> th;
        for (size_t i = 0; i < ctx->reps.size(); ++i) th.emplace_back(worker, i);
        for (auto& t : th) t.join();
    }
    for (size_t i = 0; i < ctx->reps.size(); ++i)
        if (codes[i]) return fail(ctx, codes[i], msgs[i]);
    ctx->last_e2e_ms = *std::max_element(e2e.begin(), e2e.end());
    ctx->last_kernel_ms = *std::max_element(kms.begin(), kms.end());
    ctx->last_slow_ms = *std::max_element(kslow.begin(), kslow.end());
    ctx->device_timing_pending = false;
    ctx->last_launches = 0;
    for (auto l : launches) ctx->last_launches += l;
    if (stats)
        for (auto& p : part) {
            uint64_t* d = reinterpret_cast<uint64_t*>(stats);
            const uint64_t* s = reinterpret_cast<const uint64_t*>(&p);
            for (size_t i = 0; i < sizeof(sa_stats) / 8; ++i) d[i] += s[i];
        }
    return SA_OK;
}

int sa_align_device(sa_context* ctx, const sa_params* params, const char* d_bases,
                    const uint64_t* d_offsets, uint64_t n_reads, uint64_t max_read_length,
                    sa_result* d_results, sa_stats* d_stats, void* stream) {
    if (!ctx) return fail(nullptr, SA_EINVAL, "null context");
    std::lock_guard<std::mutex> lock(ctx->mu);
    std::string why;
    if (int rc = validate_params(params, why)) return fail(ctx, rc, why);
    if (params->seed_size != ctx->seed_size)
        return fail(ctx, SA_EINVAL, "index seed size does not match params");
    if (n_reads == 0) return SA_OK;
    if (n_reads >= 0xffffffffull) return fail(ctx, SA_EINVAL, "too many reads in one batch");
    Replica& rep = ctx->reps[0];
    CUDA_TRY(ctx, cudaSetDevice(rep.device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (max_read_length == 0) return fail(ctx, SA_EINVAL, "max_read_length must be given");
    LaunchShape sh;
    if (int rc = cached_shape(rep, params, max_read_length, sh, why)) return fail(ctx, rc, why);
    if (int rc = ensure_scratch(ctx, rep, sh)) return rc;
    Stage& stg = rep.stage[kPipeStages];
    if (int rc = ensure_stage(ctx, stg, 0, n_reads)) return rc;
    const uint64_t pre_n = dev_chunk_reads() ? std::min(n_reads, dev_chunk_reads()) : n_reads;
    if (int rc = ensure_pre(ctx, stg, pre_n, sh)) return rc;
    if (int rc = ensure_gplanes(ctx, stg, sh)) return rc;  // before the per-call copy below
    // The caller's stream drives; this stage keeps only control words and
    // the seed-kernel scratch, which every call shares.  A call on another
    // stream therefore waits for the previous call's work (event `done`), so
    // calls in flight on different streams never overwrite each other's
    // cursors, records or lists.
    if (stg.done_pending) CUDA_TRY(ctx, cudaStreamWaitEvent(st, stg.done, 0));
    Stage tmp = stg;
    tmp.st = st;
    unsigned long long* stats_dst = reinterpret_cast<unsigned long long*>(d_stats);
    if (!stats_dst) stats_dst = rep.d_stats;
    uint64_t launches = 0;
    if (int rc = enqueue_align(ctx, rep, tmp, sh, d_bases, d_offsets, 0, n_reads, 0, d_results,
                               stats_dst, stg.d_overflow, true, launches))
        return rc;
    CUDA_TRY(ctx, cudaEventRecord(stg.done, st));
    stg.done_pending = true;
    ctx->last_launches = launches;
    ctx->device_timing_pending = true;
    return SA_OK;
}

int sa_last_kernel_times(sa_context* ctx, float* fast_ms, float* slow_ms) {
    if (!ctx) return fail(nullptr, SA_EINVAL, "null context");
    if (ctx->device_timing_pending) {  // events of the last sa_align_device call
        Replica& rep = ctx->reps[0];
        CUDA_TRY(ctx, cudaSetDevice(rep.device));
        float f = 0, s = 0;
        CUDA_TRY(ctx, stage_times(rep.stage[kPipeStages], f, s));
        ctx->last_kernel_ms = f;
        ctx->last_slow_ms = s;
        ctx->device_timing_pending = false;
    }
    if (fast_ms) *fast_ms = ctx->last_kernel_ms;
    if (slow_ms) *slow_ms = ctx->last_slow_ms;
    return SA_OK;
}

int sa_sync(sa_context* ctx, void* stream) {
    if (!ctx) return fail(nullptr, SA_EINVAL, "null context");
    Replica& rep = ctx->reps[0];
    CUDA_TRY(ctx, cudaSetDevice(rep.device));
    CUDA_TRY(ctx, cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    return check_errors(ctx, rep);
}

int sa_lookup_batch(sa_context* ctx, const char* seeds, uint64_t n_seeds, uint32_t* counts,
                    uint64_t* fwd_out, uint32_t* n_fwd, uint64_t* rc_out, uint32_t* n_rc,
                    uint32_t cap) {
    if (!ctx) return fail(nullptr, SA_EINVAL, "null context");
    std::lock_guard<std::mutex> lock(ctx->mu);
    if (n_seeds == 0) return SA_OK;
    if (!seeds || !counts) return fail(ctx, SA_EINVAL, "null buffer");
    if ((fwd_out == nullptr) != (rc_out == nullptr)) return fail(ctx, SA_EINVAL, "fwd_out/rc_out must both be set");
    Replica& rep = ctx->reps[0];
    CUDA_TRY(ctx, cudaSetDevice(rep.device));
    const int s = ctx->seed_size;
    char* d_seeds = nullptr;
    uint32_t *d_counts = nullptr, *d_nf = nullptr, *d_nr = nullptr;
    uint64_t *d_fwd = nullptr, *d_rc = nullptr;
    const bool lists = fwd_out != nullptr && cap > 0;
    CUDA_TRY(ctx, cudaMalloc(&d_seeds, n_seeds * s));
    CUDA_TRY(ctx, cudaMalloc(&d_counts, n_seeds * 4));
    CUDA_TRY(ctx, cudaMalloc(&d_nf, n_seeds * 4));
    CUDA_TRY(ctx, cudaMalloc(&d_nr, n_seeds * 4));
    if (lists) {
        CUDA_TRY(ctx, cudaMalloc(&d_fwd, n_seeds * cap * 8));
        CUDA_TRY(ctx, cudaMalloc(&d_rc, n_seeds * cap * 8));
    }
    CUDA_TRY(ctx, cudaMemcpy(d_seeds, seeds, n_seeds * s, cudaMemcpyHostToDevice));
    LookupLaunch a{};
    a.planes = rep.ix.planes;
    a.table = rep.ix.table;
    a.n_slots = rep.ix.n_slots;
    a.pool = rep.ix.pool;
    a.seeds = d_seeds;
    a.n_seeds = n_seeds;
    a.s = s;
    a.counts = d_counts;
    a.fwd_out = d_fwd;
    a.rc_out = d_rc;
    a.n_fwd = d_nf;
    a.n_rc = d_nr;
    a.cap = lists ? cap : 0;
    launch_lookup(a, 0);
    CUDA_TRY(ctx, cudaGetLastError());
    CUDA_TRY(ctx, cudaDeviceSynchronize());
    CUDA_TRY(ctx, cudaMemcpy(counts, d_counts, n_seeds * 4, cudaMemcpyDeviceToHost));
    if (n_fwd) CUDA_TRY(ctx, cudaMemcpy(n_fwd, d_nf, n_seeds * 4, cudaMemcpyDeviceToHost));
    if (n_rc) CUDA_TRY(ctx, cudaMemcpy(n_rc, d_nr, n_seeds * 4, cudaMemcpyDeviceToHost));
    if (lists) {
        CUDA_TRY(ctx, cudaMemcpy(fwd_out, d_fwd, n_seeds * cap * 8, cudaMemcpyDeviceToHost));
        CUDA_TRY(ctx, cudaMemcpy(rc_out, d_rc, n_seeds * cap * 8, cudaMemcpyDeviceToHost));
    }
    cudaFree(d_seeds);
    cudaFree(d_counts);
    cudaFree(d_nf);
    cudaFree(d_nr);
    if (d_fwd) cudaFree(d_fwd);
    if (d_rc) cudaFree(d_rc);
    ctx->last_launches = 1;
    return SA_OK;
}

int sa_bounded_distance_batch(const char* reads, const uint64_t* read_off, const char* windows,
                              const uint64_t* win_off, const int32_t* d_limits, uint64_t n_pairs,
                              int32_t* out, int32_t device) {
    if (n_pairs == 0) return SA_OK;
    if (!reads || !read_off || !windows || !win_off || !d_limits || !out)
        return fail(nullptr, SA_EINVAL, "null buffer");
    uint64_t mmax = 0, wmax = 0;
    int dlmax = 0;
    for (uint64_t i = 0; i < n_pairs; ++i) {
        if (d_limits[i] < 0)  // REF src/edit_distance.cpp:22-23
            return fail(nullptr, SA_EINVAL, "bounded_distance: negative d_limit");
        if (read_off[i + 1] < read_off[i] || win_off[i + 1] < win_off[i])
            return fail(nullptr, SA_EINVAL, "offsets not ascending");
        const uint64_t m = read_off[i + 1] - read_off[i];
        mmax = std::max(mmax, m);
        wmax = std::max(wmax, win_off[i + 1] - win_off[i]);
        dlmax = std::max<int>(dlmax, static_cast<int>(std::min<uint64_t>(d_limits[i], m)));
    }
    LvLaunch a{};
    a.wbr = static_cast<int>((mmax + 31) / 32 + 2);
    a.wbw = static_cast<int>((wmax + 31) / 32 + 2);
    a.f_ints = dlmax > 15 ? round4(2 * (2 * dlmax + 3)) : 0;
    a.smem_per_warp = round16(16ull * (a.wbr + a.wbw) + 4ull * a.f_ints);
    if (a.smem_per_warp > 227 * 1024) return fail(nullptr, SA_EINVAL, "pair too long for the LV kernel");
    if (cudaSetDevice(device) != cudaSuccess) return fail(nullptr, SA_ERUNTIME, "cudaSetDevice failed");
    const uint64_t rb = read_off[n_pairs] - read_off[0], wb = win_off[n_pairs] - win_off[0];
    char *d_r = nullptr, *d_w = nullptr;
    uint64_t *d_ro = nullptr, *d_wo = nullptr;
    int32_t *d_dl = nullptr, *d_out = nullptr;
    unsigned int* d_err = nullptr;
    std::vector<uint64_t> ro(read_off, read_off + n_pairs + 1), wo(win_off, win_off + n_pairs + 1);
    for (auto& v : ro) v -= read_off[0];
    for (auto& v : wo) v -= win_off[0];
#define LV_TRY(x)                                                                              \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) return fail(nullptr, SA_ERUNTIME, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)
    LV_TRY(cudaMalloc(&d_r, rb + 16));
    LV_TRY(cudaMalloc(&d_w, wb + 16));
    LV_TRY(cudaMalloc(&d_ro, (n_pairs + 1) * 8));
    LV_TRY(cudaMalloc(&d_wo, (n_pairs + 1) * 8));
    LV_TRY(cudaMalloc(&d_dl, n_pairs * 4));
    LV_TRY(cudaMalloc(&d_out, n_pairs * 4));
    LV_TRY(cudaMalloc(&d_err, 4));
    LV_TRY(cudaMemset(d_err, 0, 4));
    if (rb) LV_TRY(cudaMemcpy(d_r, reads + read_off[0], rb, cudaMemcpyHostToDevice));
    if (wb) LV_TRY(cudaMemcpy(d_w, windows + win_off[0], wb, cudaMemcpyHostToDevice));
    LV_TRY(cudaMemcpy(d_ro, ro.data(), (n_pairs + 1) * 8, cudaMemcpyHostToDevice));
    LV_TRY(cudaMemcpy(d_wo, wo.data(), (n_pairs + 1) * 8, cudaMemcpyHostToDevice));
    LV_TRY(cudaMemcpy(d_dl, d_limits, n_pairs * 4, cudaMemcpyHostToDevice));
    LV_TRY(align_set_smem(227 * 1024));
    a.reads = d_r;
    a.read_off = d_ro;
    a.wins = d_w;
    a.win_off = d_wo;
    a.d_limits = d_dl;
    a.n_pairs = static_cast<uint32_t>(n_pairs);
    a.out = d_out;
    a.error_flag = d_err;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    int warps = std::max<int>(1, std::min<int>(8, (227 * 1024) / a.smem_per_warp));
    uint64_t need_warps = std::min<uint64_t>(n_pairs, static_cast<uint64_t>(sms) * 64);
    int grid = static_cast<int>(std::max<uint64_t>(1, (need_warps + warps - 1) / warps));
    launch_lv_batch(a, grid, 32 * warps, 0);
    LV_TRY(cudaGetLastError());
    LV_TRY(cudaDeviceSynchronize());
    unsigned int err = 0;
    LV_TRY(cudaMemcpy(out, d_out, n_pairs * 4, cudaMemcpyDeviceToHost));
    LV_TRY(cudaMemcpy(&err, d_err, 4, cudaMemcpyDeviceToHost));
    cudaFree(d_r);
    cudaFree(d_w);
    cudaFree(d_ro);
    cudaFree(d_wo);
    cudaFree(d_dl);
    cudaFree(d_out);
    cudaFree(d_err);
#undef LV_TRY
    if (err) return fail(nullptr, SA_EINVAL, "bounded_distance batch: characters outside {A,C,G,T,N}");
    return SA_OK;
}

int sa_host_alloc(void** ptr, uint64_t bytes) {
    if (!ptr) return fail(nullptr, SA_EINVAL, "ptr is NULL");
    cudaError_t e = cudaMallocHost(ptr, bytes ? bytes : 1);
    if (e != cudaSuccess) return fail(nullptr, SA_ERUNTIME, cudaGetErrorString(e));
    return SA_OK;
}

void sa_host_free(void* ptr) {
    if (ptr) cudaFreeHost(ptr);
}

int sa_last_timing(const sa_context* ctx, float* e2e_ms, float* kernel_ms) {
    if (!ctx) return fail(nullptr, SA_EINVAL, "null context");
    if (e2e_ms) *e2e_ms = ctx->last_e2e_ms;
    if (kernel_ms) *kernel_ms = ctx->last_kernel_ms;
    return SA_OK;
}

int sa_last_launches(const sa_context* ctx, uint64_t* launches) {
    if (!ctx) return fail(nullptr, SA_EINVAL, "null context");
    *launches = ctx->last_launches;
    return SA_OK;
}

}  // extern "C"
