// align.cu -- the aligner hot path on sm_100a.
//
// K2..K5 of SURVEY.md §2 fused into one persistent warp-per-read kernel that
// replays Aligner::align (REF src/aligner.cpp:223-364) bit-exactly:
//   * reads are software-pipelined per warp: offsets two reads ahead in
//     registers, the next read's bytes streamed into shared memory with
//     cp.async while the current read is processed
//   * read -> 2-bit planes: SWAR decode of 4 ASCII bases per lane
//     (decode4: code arithmetic + byte_perm check), 32-base plane words assembled with shuffles; the
//     reverse complement (REF :241, genome.cpp:182-200) by __brev of planes
//   * seed offsets (REF :50-79), computed once per distinct read length
//   * seed keys + canonical probes of the HBM hash index, one lane per seed,
//     issued speculatively for 32 seeds at a time         (REF seed_index.cpp:128-143);
//     an inline (singleton) hit immediately prefetches its genome window to L2
//   * the sequential seed loop (REF :256-316): N skip, h_max filter, hits ->
//     anchors -> shared-memory vote table (single-hit fast path, otherwise
//     warp-aggregated with __match_any_sync), best-unscored selection by warp
//     argmax (REF :124-167), d_limit rule + Landau-Vishkin verification of
//     every anchor of the chosen bucket (REF :169-221), BestTracker
//     (REF :87-114), multi and pruning exits (REF :290-315)
//   * classification and result (REF :318-363)
// LV (REF src/edit_distance.cpp:19-75) is warp-cooperative: one lane per
// diagonal (registers, d_limit <= 15) or lanes striding diagonals over a
// shared-memory frontier (larger d_limit); the genome window is staged into
// shared memory once per candidate bucket and matches are extended 32 bases
// at a time by xor-ing bit planes and taking __ffs of the mismatch word.
//
// Vote tables live in shared memory (cap entries per warp).  A read whose
// candidates overflow that table is deferred to the slow kernel (same code,
// tables in global memory sized for the worst case n * h_max).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "align_kernels.cuh"
#include "common.cuh"
#include "lv.cuh"

namespace sab {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint32_t kScored = 0x80000000u;

SA_DEV uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

SA_DEV void cp_async4(void* smem_dst, const void* gsrc) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gsrc) : "memory");
}
SA_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
SA_DEV void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

SA_DEV void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// ------------------------------------------------------------------ read staging

// Decode 4 ASCII bases (byte j = base j) into nibbles: lo/hi = bits 0/1 of
// the 2-bit code (A=0 C=1 G=2 T=3, N codes as A), nn = the 'N' bytes, and
// bad != 0 when a byte is outside {A,C,G,T,N} (REF genome.cpp:182-200).
// ((c >> 1) ^ (c >> 2)) & 3 is the code of A/C/G/T; the expected character is
// looked up back from the code (byte_perm) and compared byte-wise; bits are
// gathered by one multiply per plane (no carries: the partial products are
// distinct powers of two).
SA_DEV void decode4(uint32_t v, uint32_t& lo, uint32_t& hi, uint32_t& nn, uint32_t& bad) {
    const uint32_t x = (v >> 1) ^ (v >> 2);
    lo = ((x & 0x01010101u) * 0x01020408u) >> 24;
    hi = ((x & 0x02020202u) * 0x08102040u) >> 28;
    const uint32_t t = x & 0x03030303u;
    const uint32_t sel = __byte_perm(t | (t >> 4), 0u, 0x0020u);  // nibble j = code of byte j
    const uint32_t e = __byte_perm(0x54474341u, 0u, sel);          // "ACGT"[code] per byte
    const uint32_t dn = v ^ 0x4E4E4E4Eu, de = v ^ e;
    const uint32_t nzN = ((dn & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | dn;  // bit 7 of byte j: byte j != 'N'
    const uint32_t nzE = ((de & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | de;  // bit 7 of byte j: not its ACGT char
    bad = nzN & nzE & 0x80808080u;
    nn = (((~nzN >> 7) & 0x01010101u) * 0x01020408u) >> 24;
}

// Decode a read of `len` ASCII bases whose first byte is byte `shift` of the
// 4-byte-aligned word array Wd (nwords words; generic address space: shared
// staging buffer or global) into forward planes R and reverse-complement
// planes C (REF genome.cpp:182-200), both followed by an all-N block.
// Returns true when a character outside {A,C,G,T,N} occurs (the reference
// throws from reverse_complement).
SA_DEV bool decode_read(const uint32_t* Wd, int shift, int nwords, int len, uint4* R, uint4* C,
                        int lane) {
    bool bad = false;
    const int nb = (len + 31) >> 5;
    const int rounds = (len + 127) >> 7;
    for (int rd = 0; rd < rounds; ++rd) {
        const int pos0 = rd * 128 + 4 * lane;
        uint32_t v = 0x4E4E4E4Eu;  // "NNNN"
        if (pos0 < len) {
            const int k = rd * 32 + lane;
            const uint32_t w0 = Wd[k];
            const uint32_t w1 = k + 1 < nwords ? Wd[k + 1] : 0u;
            v = __funnelshift_r(w0, w1, 8 * shift);
            const int valid = len - pos0;
            if (valid < 4) {
                const uint32_t keep = (1u << (8 * valid)) - 1u;
                v = (v & keep) | (0x4E4E4E4Eu & ~keep);
            }
        }
        uint32_t lo, hi, nn, bd;
        decode4(v, lo, hi, nn, bd);
        bad |= bd != 0u;
        const int sh = 4 * (lane & 7);
        lo <<= sh;
        hi <<= sh;
        nn <<= sh;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            lo |= __shfl_xor_sync(FULL, lo, o);
            hi |= __shfl_xor_sync(FULL, hi, o);
            nn |= __shfl_xor_sync(FULL, nn, o);
        }
        const int blk = rd * 4 + (lane >> 3);
        if ((lane & 7) == 0 && blk < nb) R[blk] = make_uint4(lo, hi, nn, 0);
    }
    if (lane == 0) R[nb] = make_uint4(0, 0, 0xFFFFFFFFu, 0);
    __syncwarp();
    // rc word q, bit b = complement of forward base len-1-32q-b
    for (int q = lane; q < nb; q += 32) {
        const int p_lo = len - 32 * (q + 1);
        uint32_t l, h, n;
        if (p_lo >= 0) {
            extract32(R, static_cast<uint64_t>(p_lo), l, h, n);
        } else {
            extract32(R, 0ull, l, h, n);
            const int s = -p_lo;
            l <<= s;
            h <<= s;
            n = (n << s) | ((1u << s) - 1u);
        }
        C[q] = make_uint4(__brev(~l), __brev(~h), __brev(n), 0);
    }
    if (lane == 0) C[nb] = make_uint4(0, 0, 0xFFFFFFFFu, 0);
    __syncwarp();
    return __any_sync(FULL, bad);
}

// Start copying a read's aligned words into a shared staging buffer.
SA_DEV void issue_read_copy(const char* src, int len, uint32_t* stage, int lane, int& shift,
                            int& nwords) {
    const uintptr_t addr = reinterpret_cast<uintptr_t>(src);
    const uintptr_t abase = addr & ~static_cast<uintptr_t>(3);
    shift = static_cast<int>(addr & 3);
    nwords = static_cast<int>((addr + static_cast<uintptr_t>(len) - abase + 3) >> 2);
    for (int w = lane; w < nwords; w += 32)
        cp_async4(stage + w, reinterpret_cast<const void*>(abase + 4ull * w));
}

// REF src/aligner.cpp:50-79 seed_offsets, restated for shift values < s <= 32:
// a tier whose shift was already used adds nothing new; otherwise it adds
// every offset shift + j*s <= max_off.  Lane 0 fills offs; returns the count.
SA_DEV int compute_offsets(int len, int s, int n, int* offs, int lane) {
    int cnt = 0;
    if (lane == 0) {
        const int max_off = len - s;
        uint32_t used = 0;
        auto emit = [&](int shift) {
            if ((used >> shift) & 1u) return;
            used |= 1u << shift;
            for (int o = shift; o <= max_off && cnt < n; o += s) offs[cnt++] = o;
        };
        emit(0);
        for (int level = 1; (1 << level) <= 4 * s && cnt < n; ++level)
            for (int odd = 1; odd < (1 << level) && cnt < n; odd += 2) emit((odd * s) >> level);
    }
    __syncwarp();
    return __shfl_sync(FULL, cnt, 0);
}

// ------------------------------------------------------------------ per-read state

struct Tracker {  // BestTracker, REF aligner.hpp:82-101
    int d_best, d_second;
    uint64_t best_pos;
    int best_dir;
};

SA_DEV void tracker_observe(Tracker& t, int merge_radius, int distance, uint64_t position,
                            int direction) {  // REF aligner.cpp:87-109
    if (t.d_best < kInfDistance && direction == t.best_dir) {
        const uint64_t delta = position > t.best_pos ? position - t.best_pos : t.best_pos - position;
        if (delta <= static_cast<uint64_t>(merge_radius)) {
            if (distance < t.d_best) {
                t.d_best = distance;
                t.best_pos = position;
            }
            return;
        }
    }
    if (distance < t.d_best) {
        t.d_second = t.d_best;
        t.d_best = distance;
        t.best_pos = position;
        t.best_dir = direction;
    } else if (distance < t.d_second) {
        t.d_second = distance;
    }
}

SA_DEV int tracker_gap(const Tracker& t) {  // REF aligner.cpp:111-114
    if (t.d_second >= kInfDistance) return kGapCap;
    return min(t.d_second - t.d_best, kGapCap);
}

struct CandTable {
    unsigned long long* ckey;   // bucket*2 + dir, insertion order
    unsigned long long* cmask;  // anchor bits
    uint32_t* ccnt;             // seeds_hitting | kScored
    uint32_t* chslot;           // hash slot of the entry (for cleanup)
    unsigned long long* hkey;   // hash keys
    uint32_t* hval;             // list index
    int cap, hcap;
};


// stats slots (sa_stats order)
enum {
    S_READS, S_TOO_SHORT, S_LOOKUPS, S_SKIP_N, S_SKIP_POP, S_ALL_POP, S_DIST, S_DIST_AFTER,
    S_EARLY_OUT, S_CELLS, S_MULTI, S_PRUNE, S_FIRST_BEST, S_SINGLE, S_MULTIPLE, S_NOT_FOUND,
    S_HITS, S_WINDOW, S_READ_BASES, S_OVERFLOW
};

struct Ctx {
    const AlignLaunch* a;
    int lane;
    int len, d_max;
    const uint4* R;
    const uint4* C;
    uint4* W;
    int* F;
    CandTable t;
    uint32_t n_cands, n_unscored;
    Tracker tr;
    uint32_t calls;
    bool first_done, first_valid;
    int first_dir;
    uint64_t first_pos;
    uint32_t cells;  // per lane, LV cells of the launch (dp_cells)
    uint32_t qf_tries, qf_hits;  // q-gram filter attempts / rejections of this warp
    uint32_t* qbm;               // its 4^kQfQ-bit bitmap (shared memory), null: no filter
    // Per-read counters, lane-distributed: lane k holds stats slot k (sa_stats
    // order) for the read in flight -- one register for all of them.  Added to
    // the warp totals when the read completes, dropped if it overflows.
    uint32_t rs;
};

SA_DEV void stat_add(Ctx& x, int slot, uint32_t v) { x.rs += x.lane == slot ? v : 0u; }

// Slot of a candidate key (bucket << 1 | dir, < 2^33) in the candidate hash
// index: 32-bit multiplicative hash, high half rotated down.  Only placement
// depends on it; candidate order is the insertion order (REF aligner.cpp:124-134).
SA_DEV uint32_t cand_hash(unsigned long long key, int hcap) {
    const uint32_t h = static_cast<uint32_t>(key) * 0x9E3779B1u + static_cast<uint32_t>(key >> 32) * 0x85EBCA77u;
    return __funnelshift_l(h, h, 16) & static_cast<uint32_t>(hcap - 1);
}

// Warp-cooperative add_hit for up to 32 hits (REF aligner.cpp:124-134).
// Returns false when the table would overflow.
SA_DEV bool insert_wave(Ctx& x, bool valid, unsigned long long key, int bit) {
    const int lane = x.lane;
    const uint32_t vmask = __ballot_sync(FULL, valid);
    if (vmask == 0) return true;
    if ((vmask & (vmask - 1)) == 0) {  // one hit: uniform probe, no atomics
        const int src = __ffs(vmask) - 1;
        key = __shfl_sync(FULL, key, src);
        bit = __shfl_sync(FULL, bit, src);
        uint32_t h = cand_hash(key, x.t.hcap);
        for (;;) {
            const unsigned long long cur = x.t.hkey[h];
            if (cur == key) {
                const uint32_t idx = x.t.hval[h];
                if (lane == 0) {
                    x.t.ccnt[idx] += 1u;
                    x.t.cmask[idx] |= 1ull << bit;
                }
                break;
            }
            if (cur == kEmptyKey) {
                if (x.n_cands + 1 > static_cast<uint32_t>(x.t.cap)) return false;
                const uint32_t idx = x.n_cands;
                if (lane == 0) {
                    x.t.hkey[h] = key;
                    x.t.hval[h] = idx;
                    x.t.chslot[idx] = h;
                    x.t.ckey[idx] = key;
                    x.t.cmask[idx] = 1ull << bit;
                    x.t.ccnt[idx] = 1u;
                }
                x.n_cands += 1;
                x.n_unscored += 1;
                break;
            }
            h = (h + 1) & static_cast<uint32_t>(x.t.hcap - 1);
        }
        __syncwarp();
        return true;
    }
    const unsigned long long ukey = valid ? key : (0xFFFFFFFF00000000ull | static_cast<unsigned>(lane));
    const unsigned peers = __match_any_sync(FULL, ukey);
    const int leader = __ffs(peers) - 1;
    const bool is_leader = valid && lane == leader;
    bool isnew = false;
    uint32_t slot = 0, idx = 0;
    if (is_leader) {
        uint32_t h = cand_hash(key, x.t.hcap);
        volatile unsigned long long* hk = x.t.hkey;
        for (;;) {
            unsigned long long cur = hk[h];
            if (cur == key) {
                idx = x.t.hval[h];
                break;
            }
            if (cur == kEmptyKey) {
                unsigned long long old = atomicCAS(x.t.hkey + h, kEmptyKey, key);
                if (old == kEmptyKey) {
                    isnew = true;
                    slot = h;
                    break;
                }
                if (old == key) {
                    idx = x.t.hval[h];
                    break;
                }
            }
            h = (h + 1) & static_cast<uint32_t>(x.t.hcap - 1);
        }
    }
    const uint32_t newmask = __ballot_sync(FULL, isnew);
    const uint32_t nnew = __popc(newmask);
    if (x.n_cands + nnew > static_cast<uint32_t>(x.t.cap)) return false;
    if (isnew) {
        idx = x.n_cands + __popc(newmask & lanemask_lt());
        x.t.hval[slot] = idx;
        x.t.chslot[idx] = slot;
        x.t.ckey[idx] = key;
        x.t.cmask[idx] = 0ull;
        x.t.ccnt[idx] = 0u;
    }
    x.n_cands += nnew;
    x.n_unscored += nnew;
    __syncwarp();
    idx = __shfl_sync(FULL, idx, leader);
    if (is_leader) x.t.ccnt[idx] += static_cast<uint32_t>(__popc(peers));
    if (valid) {
        if (peers == (1u << lane)) x.t.cmask[idx] |= 1ull << bit;
        else atomicOr(x.t.cmask + idx, 1ull << bit);
    }
    __syncwarp();
    return true;
}

#ifndef SA_PB_SEG
#define SA_PB_SEG 0
#endif
#ifndef SA_QGRAM_FILTER
#define SA_QGRAM_FILTER 1  // long-read LVs: the exact q-gram pre-test (lv.cuh qgram_reject); 0 off
#endif
#ifndef SA_MASK_LV
#define SA_MASK_LV 0  // 1: the mask LV (lv.cuh lv_seg) scores reads <= 128 bases in the warp kernel (measured slower, see DESIGN)
#endif

SA_DEV unsigned long long shfl64(unsigned long long v, int src) {
    const uint32_t lo = __shfl_sync(FULL, static_cast<uint32_t>(v), src);
    const uint32_t hi = __shfl_sync(FULL, static_cast<uint32_t>(v >> 32), src);
    return (static_cast<unsigned long long>(hi) << 32) | lo;
}

// REF aligner.cpp:169-221 score_candidate
// kSys: the kernel may run the systolic long-read LV (lv_sys): only the
// dynamic-fetch kernel of reads > 1 kbp; elsewhere its inlined code only
// raised register pressure (C3's seeded kernel spilled 40 -> 112 B, 120 -> 140 ms)
template <bool kRegLV, bool kSys = false>
SA_DEV void score_candidate(Ctx& x, uint32_t idx) {
    const AlignLaunch& a = *x.a;
    const int lane = x.lane;
    const unsigned long long kk = x.t.ckey[idx];
    const unsigned long long mm = x.t.cmask[idx];
    __syncwarp();
    if (lane == 0) x.t.ccnt[idx] |= kScored;
    x.n_unscored--;

    const int c = a.c, d_max = x.d_max;
    int d_limit;
    if (x.tr.d_best > d_max) d_limit = d_max + c - 1;
    else if (x.tr.d_second >= x.tr.d_best + c) d_limit = x.tr.d_best + c - 1;
    else d_limit = x.tr.d_best - 1;
    if (a.force) d_limit = d_max + c - 1;
    if (d_limit < 0) return;  // (:184)

    const int dir = static_cast<int>(kk & 1ull);
    const uint64_t base_pos = (kk >> 1) * static_cast<uint64_t>(a.bs);
    const uint64_t amin = base_pos + static_cast<uint64_t>(__ffsll(static_cast<long long>(mm)) - 1);
    const uint64_t amax = base_pos + static_cast<uint64_t>(63 - __clzll(static_cast<long long>(mm)));
    const uint4* orient = dir ? x.C : x.R;

    // Register LV (d_limit <= 15): the LV reads the genome planes in global
    // memory through L1 (the window was prefetched into L2 when the seed hit
    // was found); C1 494 -> 503 M reads/s, C2 194 -> 203 M.  The shared-memory
    // LV (long reads, many steps per window) keeps the staged union of the
    // bucket's windows (REF genome.cpp:114-123 substring: truncated at the
    // genome end only): global reads measured 6-8% slower there.
    uint64_t gb0 = 0;
    const uint4* Wsrc = a.planes;
    if (!kRegLV && !a.gw) {
        gb0 = amin >> 5;
        uint64_t end = amax + static_cast<uint64_t>(x.len) + static_cast<uint64_t>(d_limit);
        if (end > a.glen) end = a.glen;
        if (amin < a.glen) {
            const int nblk = static_cast<int>(((end - 1) >> 5) - gb0) + 2;
            for (int t = lane; t < nblk; t += 32) x.W[t] = __ldg(a.planes + gb0 + t);
        }
        __syncwarp();
        Wsrc = x.W;
    }

    int best_d = kInfDistance;
    uint64_t best_anchor = 0;
#if SA_MASK_LV
    if (kRegLV && x.len <= kMaskMaxLen) {
        // mask LV (lv_seg): the bucket's anchors in segments of 2 d_limit + 1
        // lanes, as many per pass as fit, in ascending order
        const int wd = 2 * d_limit + 1, per = 32 / wd, seg = lane / wd;
        const uint64_t nbg = (a.glen + 31) >> 5;
        for (unsigned long long m = mm; m != 0ull;) {
            unsigned long long mi = m;
            for (int t = 0; t < seg && mi != 0ull; ++t) mi &= mi - 1ull;
            const bool live = seg < per && mi != 0ull;
            const uint64_t anchor = base_pos + static_cast<uint64_t>(__ffsll(static_cast<long long>(mi)) - 1);
            const bool valid = live && anchor < a.glen;
            int w = 0;
            if (valid) {
                const uint64_t rem = a.glen - anchor;
                const uint64_t want = static_cast<uint64_t>(x.len) + static_cast<uint64_t>(d_limit);
                w = static_cast<int>(want < rem ? want : rem);
            }
            const int d = lv_seg(orient, x.len, a.planes, nbg, anchor, w, valid, d_limit, lane, x.cells);
            // per anchor, in order: one call each (REF aligner.cpp:193-210)
            const bool leader = valid && lane == seg * wd;
            const uint32_t vm = __ballot_sync(FULL, leader);
            if (vm) {
                const uint32_t em = __ballot_sync(FULL, leader && d < 0);
                const uint32_t nv = __popc(vm);
                uint32_t na = nv, ne = __popc(em);
                if (x.calls == 0) {  // the read's first call is not "after first"
                    --na;
                    if (em & (vm & (0u - vm))) --ne;
                }
                stat_add(x, S_DIST, nv);
                stat_add(x, S_DIST_AFTER, na);
                stat_add(x, S_EARLY_OUT, ne);
                stat_add(x, S_WINDOW, __reduce_add_sync(FULL, leader ? static_cast<uint32_t>(w) : 0u));
                x.calls += nv;
                const uint32_t kb = __reduce_min_sync(FULL, leader && d >= 0 ? (static_cast<uint32_t>(d) << 8) | lane
                                                                            : 0xffffffffu);
                if (kb != 0xffffffffu && static_cast<int>(kb >> 8) < best_d) {  // earlier passes win ties
                    best_d = static_cast<int>(kb >> 8);
                    best_anchor = shfl64(anchor, static_cast<int>(kb & 0xffu));
                }
            }
            for (int t = 0; t < per && m != 0ull; ++t) m &= m - 1ull;
        }
    } else
#endif
    for (unsigned long long m = mm; m != 0ull; m &= m - 1ull) {
        const uint64_t anchor = base_pos + static_cast<uint64_t>(__ffsll(static_cast<long long>(m)) - 1);
        if (anchor >= a.glen) continue;
        const uint64_t rem = a.glen - anchor;
        const uint64_t want = static_cast<uint64_t>(x.len) + static_cast<uint64_t>(d_limit);
        const int w = static_cast<int>(want < rem ? want : rem);
        const uint32_t wofs = static_cast<uint32_t>(anchor - gb0 * 32);
        int d;
        // long-read LVs: the q-gram filter first (lv.cuh qgram_reject) where the
        // warp has a bitmap (x.qbm: the LV frontier area, >= 512 B), where a
        // piece's band is at most ~2 pieces wide (d_limit <= kQfPiece: its cost
        // per read q-gram is (piece + 2 d_limit) / piece inserts; C4's 607
        // measured 77 -> 91 ms with nothing rejected) and, per warp, while it
        // keeps paying off (no more tries after 32 attempts with < 1/8
        // rejected).  Not in the register-LV (short-read) kernels: there it
        // would reject ~90% of the seed loop's failing LVs, but its code cost
        // the C2 warp kernel 32 B of spills and C2 432 -> 420 M reads/s.
        if (!kRegLV && SA_QGRAM_FILTER && x.qbm != nullptr && d_limit <= kQfPiece &&
            (x.qf_tries < 32 || 8 * x.qf_hits >= x.qf_tries) &&
            (++x.qf_tries, qgram_reject(orient, x.len, Wsrc, wofs, w, d_limit, x.qbm, lane))) {
            ++x.qf_hits;
            d = -1;
        } else {
            d = lv_warp<kRegLV, kSys>(orient, x.len, Wsrc, wofs, w, d_limit, x.F, lane, x.cells, a.f16 != 0);
        }
#if SA_DEBUG_COUNTERS
        if (a.dbg && lane == 0) {  // seed-loop (warp) LV: calls, iterations, d_limit sum
            atomicAdd(a.dbg + 4, 1u);
            atomicAdd(a.dbg + 5, static_cast<unsigned>(d >= 0 ? d + 1 : d_limit + 1));
            atomicAdd(a.dbg + 6, static_cast<unsigned>(d_limit));
        }
#endif
        stat_add(x, S_DIST, 1u);
        x.calls++;
        stat_add(x, S_WINDOW, static_cast<uint32_t>(w));
        if (x.calls > 1) {
            stat_add(x, S_DIST_AFTER, 1u);
            if (d < 0) stat_add(x, S_EARLY_OUT, 1u);
        }
        if (d >= 0 && d < best_d) {
            best_d = d;
            best_anchor = anchor;
        }
    }
    if (!x.first_done) {
        x.first_done = true;
        if (best_d < kInfDistance) {
            x.first_valid = true;
            x.first_pos = best_anchor;
            x.first_dir = dir;
        }
    }
    if (best_d < kInfDistance) tracker_observe(x.tr, a.bs, best_d, best_anchor, dir);
}

// REF aligner.cpp:141-167 score_best_candidate's choice: the unscored
// candidate with most seeds hitting, then smallest anchor, then Forward.
// Returns its index, -1 when nothing is unscored.
SA_DEV int pick_best(Ctx& x) {
    if (x.n_unscored == 0) return -1;
    if (x.n_cands == 1) return 0;  // the only candidate is the unscored one
    const AlignLaunch& a = *x.a;
    uint32_t bc = 0;
    unsigned long long bk = ~0ull;
    int bi = -1;
    for (uint32_t j = x.lane; j < x.n_cands; j += 32) {
        const uint32_t cc = x.t.ccnt[j];
        if (cc & kScored) continue;
        const unsigned long long kk = x.t.ckey[j];
        const unsigned long long mm = x.t.cmask[j];
        const unsigned long long amin = (kk >> 1) * static_cast<unsigned long long>(a.bs) +
                                        static_cast<unsigned long long>(__ffsll(static_cast<long long>(mm)) - 1);
        const unsigned long long ord = (amin << 1) | (kk & 1ull);
        if (cc > bc || (cc == bc && ord < bk)) {
            bc = cc;
            bk = ord;
            bi = static_cast<int>(j);
        }
    }
    // warp argmax of (seeds_hitting, then smallest (amin, dir)) with three
    // single-instruction reductions instead of a 5-step shuffle tree of
    // three values (score_best was 18% of the warp kernel at C2)
    const uint32_t mc = __reduce_max_sync(FULL, bc);
    const bool in = bi >= 0 && bc == mc;
    const uint32_t khi = static_cast<uint32_t>(bk >> 32), klo = static_cast<uint32_t>(bk);
    const uint32_t mhi = __reduce_min_sync(FULL, in ? khi : 0xffffffffu);
    const uint32_t mlo = __reduce_min_sync(FULL, in && khi == mhi ? klo : 0xffffffffu);
    const uint32_t win = __ballot_sync(FULL, in && khi == mhi && klo == mlo);
    if (win == 0u) return -1;  // nothing unscored
    return __shfl_sync(FULL, bi, __ffs(win) - 1);
}

template <bool kRegLV, bool kSys = false>
SA_DEV void score_best(Ctx& x) {
    const int bi = pick_best(x);
    if (bi >= 0) score_candidate<kRegLV, kSys>(x, static_cast<uint32_t>(bi));
}

// ------------------------------------------------------------------ pruning batch
// The pruning loop (REF aligner.cpp:296-315) scores every remaining unscored
// candidate, best first, each under a d_limit re-derived from the tracker.
// No hit is added in that loop, so the order is fixed; and every d_limit it
// can derive is at most B = d_best + c - 1 (d_best <= d_max: d_best only
// falls, and a refined best keeps d_limit below the old d_best + c - 1; with
// d_best > d_max or force_max_dlimit, B = d_max + c - 1).  A bounded distance
// is exact when it is <= the bound (REF edit_distance.cpp:19-75; a longer
// window never changes a value <= d_limit), so the
// batch runs the LVs of up to 64 anchors of the next candidates (in selection
// order) at once -- one anchor per lane, the thread-serial wavefront at bound
// B -- and then replays the loop candidate by candidate: d_limit from the
// tracker, each anchor's value cut at d_limit, calls / early-out / window
// counters per anchor in order, min with the earliest anchor on ties, one
// observe, the multi exit.  Same results and counters as scoring them one by
// one (dp_cells aside, which is implementation-specific).
// Shared memory per warp: the lanes' frontiers [kPbF][32] shorts, 64 slot
// entries (candidate of the batch, anchor bit), and the selection order.
#ifndef SA_PRUNE_BATCH
#define SA_PRUNE_BATCH 1
#endif
constexpr int kPbMax = 5;                // largest bound B the batch takes
constexpr int kPbF = 2 * kPbMax + 3;     // frontier entries per lane
constexpr uint32_t kPbBytes = kPbF * 32 * 2 + 64 * 4;  // 1088, a multiple of 16

// Selection order of the unscored candidates (the table holds <= 64):
// bitonic sort of 64 keys, two per lane, on (seeds_hitting desc, amin asc,
// Forward first) -- the order score_best_candidate's repeated argmax takes
// (REF aligner.cpp:141-167) when nothing changes the counts.  order[p] =
// candidate index at position p.  Returns false (nothing written) when a
// count does not fit the key.
SA_DEV bool select_order(Ctx& x, uint8_t* order) {
    const AlignLaunch& a = *x.a;
    const int lane = x.lane;
    unsigned long long v[2];
    bool ok = true;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t j = 2 * lane + h;
        v[h] = ~0ull;
        if (j < x.n_cands) {
            const uint32_t cc = x.t.ccnt[j];
            if (!(cc & kScored)) {
                ok &= cc < 0xffffu;
                const unsigned long long kk = x.t.ckey[j];
                const unsigned long long amin =
                    (kk >> 1) * static_cast<unsigned long long>(a.bs) +
                    static_cast<unsigned long long>(__ffsll(static_cast<long long>(x.t.cmask[j])) - 1);
                v[h] = (static_cast<unsigned long long>(0xffffu - cc) << 48) | (amin << 7) | ((kk & 1ull) << 6) | j;
            }
        }
    }
    if (!__all_sync(FULL, ok)) return false;
    if (x.n_cands <= 32) {  // one key per lane, a 32-key network (candidate l from lane l / 2)
        const unsigned long long a0 = shfl64(v[0], lane >> 1), a1 = shfl64(v[1], lane >> 1);
        unsigned long long u = (lane & 1) ? a1 : a0;
#pragma unroll 1
        for (int k = 2; k <= 32; k <<= 1) {
            const bool up = (lane & k) == 0;
#pragma unroll 1
            for (int j = k >> 1; j > 0; j >>= 1) {
                const unsigned long long o = shfl64(u, lane ^ j);
                u = (((lane & j) == 0) == up) ? min(u, o) : max(u, o);
            }
        }
        order[lane] = static_cast<uint8_t>(u & 63u);
        __syncwarp();
        return true;
    }
    // rolled loops: every warp entering the pruning loop runs this, and the
    // unrolled network's ~1k instructions measured as instruction-fetch
    // stalls (33% of the warp kernel's samples at C2)
#pragma unroll 1
    for (int k = 2; k <= 64; k <<= 1) {
        const bool up = ((2 * lane) & k) == 0;
#pragma unroll 1
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == 1) {
                const unsigned long long lo = min(v[0], v[1]), hi = max(v[0], v[1]);
                v[0] = up ? lo : hi;
                v[1] = up ? hi : lo;
            } else {
                const int pl = lane ^ (j >> 1);
                const bool keep_min = ((lane & (j >> 1)) == 0) == up;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const unsigned long long o = shfl64(v[h], pl);
                    v[h] = keep_min ? min(v[h], o) : max(v[h], o);
                }
            }
        }
    }
    order[2 * lane] = static_cast<uint8_t>(v[0] & 63u);
    order[2 * lane + 1] = static_cast<uint8_t>(v[1] & 63u);
    __syncwarp();
    return true;
}

// The same order for larger tables (the global-table kernel: up to 16 k
// candidates), sorted in place in the table's hash-value area -- free once
// no more hits are added; hcap >= 2 cap gives room for next_pow2(n) keys --
// by a warp bitonic network in memory.  keys[p] & 0x3fff = candidate index
// at position p.  Returns false when a count or the index does not fit.
SA_DEV bool select_order_large(Ctx& x, unsigned long long* keys) {
    const AlignLaunch& a = *x.a;
    const int lane = x.lane;
    const uint32_t n = x.n_cands;
    if (n > 0x4000u) return false;
    uint32_t P = 64;
    while (P < n) P <<= 1;
    bool ok = true;
    for (uint32_t j = lane; j < P; j += 32) {
        unsigned long long v = ~0ull;
        if (j < n) {
            const uint32_t cc = x.t.ccnt[j];
            if (!(cc & kScored)) {
                ok &= cc < 0xffffu;
                const unsigned long long kk = x.t.ckey[j];
                const unsigned long long amin =
                    (kk >> 1) * static_cast<unsigned long long>(a.bs) +
                    static_cast<unsigned long long>(__ffsll(static_cast<long long>(x.t.cmask[j])) - 1);
                v = (static_cast<unsigned long long>(0xffffu - cc) << 48) | (amin << 15) | ((kk & 1ull) << 14) | j;
            }
        }
        keys[j] = v;
    }
    if (!__all_sync(FULL, ok)) return false;
    __syncwarp();
    for (uint32_t k = 2; k <= P; k <<= 1) {
        for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
            for (uint32_t i = lane; i < P / 2; i += 32) {
                const uint32_t lo = ((i & ~(jj - 1u)) << 1) | (i & (jj - 1u)), hi = lo + jj;  // jj: power of two
                const bool up = (lo & k) == 0;
                const unsigned long long u = keys[lo], v = keys[hi];
                if ((u > v) == up) {
                    keys[lo] = v;
                    keys[hi] = u;
                }
            }
            __syncwarp();
        }
    }
    return true;
}

// The whole rest of the pruning loop.  Returns true when the multi exit fired.
SA_DEV bool prune_all(Ctx& x, unsigned char* pb, int B) {
    const AlignLaunch& a = *x.a;
    const int lane = x.lane;
    short* PF = reinterpret_cast<short*>(pb);
    uint8_t* slot_c = pb + kPbF * 32 * 2;  // slot -> candidate of the batch
    uint8_t* slot_b = slot_c + 64;          // slot -> anchor bit
    uint8_t* order = slot_b + 64;           // selection order (tables of <= 64)
    int8_t* slot_d = reinterpret_cast<int8_t*>(order + 64);  // slot -> distance (mask LV passes)
#if SA_PB_SEG
    const bool seg_lv = a.pb_on == 2 && x.len <= kMaskMaxLen;
#else
    constexpr bool seg_lv = false;  // SA_PB_SEG=1 builds the mask-LV batch (pb_on == 2; measured slower)
#endif
    const bool sorted = x.n_cands <= 64 && select_order(x, order);
    // larger tables (global-table kernel): sorted in the hash-value area
    unsigned long long* big = (!sorted && x.n_cands > 64 && x.t.hcap >= 2 * x.t.cap)
                                  ? reinterpret_cast<unsigned long long*>(x.t.hval)
                                  : nullptr;
    if (big && !select_order_large(x, big)) big = nullptr;
    const int c = a.c, d_max = x.d_max;
    uint32_t pos = 0;  // next position in the selection order
    while (x.n_unscored > 0) {
        // 1. the next candidates in selection order, up to 32 candidates and
        //    64 anchors; lane j holds the j-th
        int my_idx = 0, nc = 0;
        uint32_t my_cnt = 0, my_start = 0;
        if (sorted || big) {
            const uint32_t p = pos + lane;
            const bool have = p < pos + x.n_unscored;
            if (have) {
                my_idx = sorted ? order[p] : static_cast<int>(big[p] & 0x3fffu);
                my_cnt = __popcll(static_cast<long long>(x.t.cmask[my_idx]));
            }
            my_start = my_cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(FULL, my_start, o);
                if (lane >= o) my_start += t;
            }
            nc = __popc(__ballot_sync(FULL, have && my_start <= 64));  // my_start is the inclusive end here
            my_start -= my_cnt;
            if (lane < nc) x.t.ccnt[my_idx] |= kScored;
            __syncwarp();
            pos += nc;
        } else {  // repeated argmax (larger tables: the global-table kernel)
            int ns = 0;
            while (nc < 32 && x.n_unscored > static_cast<uint32_t>(nc)) {
                const int bi = pick_best(x);
                const int na = __popcll(static_cast<long long>(x.t.cmask[bi]));
                if (ns + na > 64) break;
                if (lane == nc) {
                    my_idx = bi;
                    my_cnt = static_cast<uint32_t>(na);
                    my_start = static_cast<uint32_t>(ns);
                }
                __syncwarp();
                if (lane == 0) x.t.ccnt[bi] |= kScored;
                __syncwarp();
                ++nc;
                ns += na;
            }
        }
        x.n_unscored -= nc;
        const unsigned long long my_key = x.t.ckey[my_idx];
        const uint32_t ns = __shfl_sync(FULL, my_start + my_cnt, nc - 1);
        if (lane < nc) {
            uint32_t sl = my_start;
            for (unsigned long long m = x.t.cmask[my_idx]; m != 0ull; m &= m - 1ull, ++sl) {
                slot_c[sl] = static_cast<uint8_t>(lane);
                slot_b[sl] = static_cast<uint8_t>(__ffsll(static_cast<long long>(m)) - 1);
            }
        }
        __syncwarp();
        // 2. one anchor per lane (two passes when the batch holds more than 32),
        //    or (pb_on == 2) mask-LV passes of 2B + 1 lanes per anchor
        int dist[2] = {-1, -1};
        uint32_t cand[2] = {0xffu, 0xffu}, rem[2] = {0, 0};
        bool valid[2] = {false, false};
        if (seg_lv) {
            const int wd = 2 * B + 1, per = 32 / wd, seg = lane / wd;
            const uint64_t nbg = (a.glen + 31) >> 5;
            for (uint32_t s0 = 0; s0 < ns; s0 += per) {
                const uint32_t sl = s0 + seg;
                const bool live = seg < per && sl < ns;
                const int j = live ? slot_c[sl] : 0;
                const unsigned long long kk = __shfl_sync(FULL, my_key, j);
                const uint64_t anchor = (kk >> 1) * static_cast<uint64_t>(a.bs) + (live ? slot_b[sl] : 0);
                const bool ok = live && anchor < a.glen;
                int w = 0;
                if (ok) {
                    const uint64_t rm = a.glen - anchor;
                    const uint64_t want = static_cast<uint64_t>(x.len) + static_cast<uint64_t>(B);
                    w = static_cast<int>(want < rm ? want : rm);
                }
                const int d = lv_seg((kk & 1ull) ? x.C : x.R, x.len, a.planes, nbg, anchor, w, ok, B, lane, x.cells);
                if (ok && lane == seg * wd) slot_d[sl] = static_cast<int8_t>(d);
            }
            __syncwarp();
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t sl = lane + 32 * h;
            const int j = sl < ns ? slot_c[sl] : 0;
            const unsigned long long kk = __shfl_sync(FULL, my_key, j);
            if (sl < ns) {
                cand[h] = static_cast<uint32_t>(j);
                const uint64_t anchor = (kk >> 1) * static_cast<uint64_t>(a.bs) + slot_b[sl];
                if (anchor < a.glen) {
                    valid[h] = true;
                    const uint64_t rm = a.glen - anchor;
                    rem[h] = rm < 0xffffffffull ? static_cast<uint32_t>(rm) : 0xffffffffu;
                    if (seg_lv) {
                        dist[h] = slot_d[sl];
                    } else {
                        const uint64_t want = static_cast<uint64_t>(x.len) + static_cast<uint64_t>(B);
                        const int w = static_cast<int>(want < rm ? want : rm);
                        dist[h] = lv_thread((kk & 1ull) ? x.C : x.R, x.len, a.planes, static_cast<uint32_t>(anchor), w,
                                            B, PF + lane, 32, x.cells, B);
                    }
                }
            }
        }
        // 3. replay (uniform control).  Between two candidates that observe
        // something the tracker -- and so d_limit -- is constant, and a
        // candidate none of whose anchors is within d_limit only moves
        // counters: such runs are applied in bulk.
        int j0 = 0;
        while (j0 < nc) {
            int d_limit;  // REF aligner.cpp:176-183
            if (x.tr.d_best > d_max) d_limit = d_max + c - 1;
            else if (x.tr.d_second >= x.tr.d_best + c) d_limit = x.tr.d_best + c - 1;
            else d_limit = x.tr.d_best - 1;
            if (a.force) d_limit = d_max + c - 1;
            if (d_limit < 0) {  // (:184) scored, nothing else (not even first_scored_done_); then the multi check
                ++j0;
                if (x.tr.d_best < c && x.tr.d_second < x.tr.d_best + c) return true;
                continue;
            }
            // first candidate (from j0) with an anchor within d_limit
            uint32_t jh = static_cast<uint32_t>(nc);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const bool hit = valid[h] && cand[h] >= static_cast<uint32_t>(j0) && dist[h] >= 0 && dist[h] <= d_limit;
                jh = min(jh, __reduce_min_sync(FULL, hit ? cand[h] : 0xffu));
            }
            // candidates j0 .. jh (jh included when < nc): their anchors' calls
            // in order; only the read's very first call is not "after first"
            // (REF aligner.cpp:196-205)
            uint32_t nv = 0, ne = 0, wsum = 0, keyv = 0xffffffffu, firstv = 0xffffffffu;
            bool mine[2], early[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t sl = lane + 32 * h;
                mine[h] = valid[h] && cand[h] >= static_cast<uint32_t>(j0) && cand[h] <= jh;
                const bool in_lim = mine[h] && dist[h] >= 0 && dist[h] <= d_limit;
                early[h] = mine[h] && !in_lim;
                nv += __popc(__ballot_sync(FULL, mine[h]));
                ne += __popc(__ballot_sync(FULL, early[h]));
                if (mine[h]) {
                    const uint32_t want = static_cast<uint32_t>(x.len + d_limit);
                    wsum += want < rem[h] ? want : rem[h];
                    firstv = min(firstv, sl);
                    if (in_lim) keyv = min(keyv, (static_cast<uint32_t>(dist[h]) << 8) | sl);
                }
            }
            if (nv > 0) {
                uint32_t na = nv;
                if (x.calls == 0) {  // the first of these calls is the read's first
                    const uint32_t fs = __reduce_min_sync(FULL, firstv);
                    --na;
                    if (__any_sync(FULL, (early[0] && static_cast<uint32_t>(lane) == fs) ||
                                             (early[1] && static_cast<uint32_t>(lane + 32) == fs)))
                        --ne;
                }
                stat_add(x, S_DIST, nv);
                stat_add(x, S_DIST_AFTER, na);
                stat_add(x, S_EARLY_OUT, ne);
                stat_add(x, S_WINDOW, __reduce_add_sync(FULL, wsum));
                x.calls += nv;
            }
            if (!x.first_done && jh > static_cast<uint32_t>(j0)) x.first_done = true;  // first scored: nothing within
            if (jh >= static_cast<uint32_t>(nc)) break;
            // candidate jh: min distance, earliest anchor on ties, one observe
            const uint32_t best = __reduce_min_sync(FULL, keyv);
            const unsigned long long kk = __shfl_sync(FULL, my_key, static_cast<int>(jh));
            const int dir = static_cast<int>(kk & 1ull);
            const uint64_t anchor = (kk >> 1) * static_cast<uint64_t>(a.bs) + slot_b[best & 0xffu];
            if (!x.first_done) {
                x.first_done = true;
                x.first_valid = true;
                x.first_pos = anchor;
                x.first_dir = dir;
            }
            tracker_observe(x.tr, a.bs, static_cast<int>(best >> 8), anchor, dir);
            if (x.tr.d_best < c && x.tr.d_second < x.tr.d_best + c) return true;  // REF :307-312
            j0 = static_cast<int>(jh) + 1;
        }
        __syncwarp();
    }
    return false;
}

SA_DEV void clear_table(CandTable& t, uint32_t n_cands, bool full, int lane) {
    __syncwarp();
    if (full) {
        for (int j = lane; j < t.hcap; j += 32) t.hkey[j] = kEmptyKey;
    } else {
        for (uint32_t j = lane; j < n_cands; j += 32) t.hkey[t.chslot[j]] = kEmptyKey;
    }
    __syncwarp();
}

// per-seed flags
constexpr uint32_t kSeedN = 1, kSeedQflip = 2, kSeedPal = 4, kSeedSingleRc = 8;
// A seed the seed kernel left unprobed (beyond its eager count): the record
// holds the canonical key in .y (low) / .z (high) until resolve_lazy probes it.
constexpr uint32_t kSeedLazy = 16;

// Probe a lazy record's key (REF seed_index.cpp:128-143), giving the record
// the seed kernel would have written.
SA_DEV uint4 resolve_lazy(const AlignLaunch& a, uint4 rec) {
    const uint64_t canon = (static_cast<uint64_t>(rec.z) << 32) | rec.y;
    uint32_t fl = rec.x & ~kSeedLazy;
    unsigned pl = 0, m = 0;
    const bool found = probe_slot(a.table, a.n_slots, canon, pl, m);
    uint32_t c = 0;
    if (found) {
        const uint32_t ntot = m & 0x7fffffffu;
        c = (fl & kSeedPal) ? 2u * ntot : ntot;
        if (m & 0x80000000u) fl |= kSeedSingleRc;
    }
    return make_uint4(fl, c, found ? pl : 0u, rec.w);
}


// Seed at read offset `off` (planes R): flags (N / query-is-rc-of-canon /
// palindrome) and its canonical planar key.
SA_DEV uint32_t seed_key(const AlignLaunch& a, const uint4* R, int off, uint64_t& canon) {
    uint32_t lo, hi, nn;
    extract32(R, static_cast<uint64_t>(off), lo, hi, nn);
    canon = 0;
    if (nn & seed_mask32(a.s)) return kSeedN;  // REF aligner.cpp:259-262
    const uint64_t key = planar_key(lo, hi, a.s);
    const uint64_t rc = planar_rc_key(lo, hi, a.s);
    canon = key < rc ? key : rc;
    uint32_t f = 0;
    if (key != canon) f |= kSeedQflip;
    if (key == rc) f |= kSeedPal;
    return f;
}

// Seed record {flags, hit count (REF LookupResult::count), payload, offset}
// from a resolved probe.  A singleton hit is the likely candidate: its genome
// window is prefetched into L2 right away.
SA_DEV uint4 seed_record(const AlignLaunch& a, uint32_t flags, bool found, unsigned payload,
                         unsigned meta, int off, int len) {
    uint32_t cnt = 0;
    if (found) {
        const uint32_t ntot = meta & 0x7fffffffu;
        cnt = (flags & kSeedPal) ? 2u * ntot : ntot;
        if (meta & 0x80000000u) flags |= kSeedSingleRc;
        if (ntot == 1 && !(flags & kSeedPal)) {
            const uint32_t dir = ((meta >> 31) & 1u) ^ ((flags & kSeedQflip) ? 1u : 0u);
            const int64_t anc = static_cast<int64_t>(payload) - (dir ? (len - a.s - off) : off);
            const uint64_t b = anc < 0 ? 0 : (static_cast<uint64_t>(anc) >> 5);
            prefetch_l2(a.planes + b);
            prefetch_l2(a.planes + b + ((len + a.dl_max + 32) >> 5));
        }
    }
    return make_uint4(flags, cnt, found ? payload : 0u, static_cast<uint32_t>(off));
}

// Probe seeds i .. i+31 synchronously (one lane each) into recs[0..31].
SA_DEV void compute_wave_sync(const AlignLaunch& a, const uint4* R, const int* offs, int i,
                              int n_eff, int len, uint4* recs, int lane) {
    const int si = i + lane;
    if (si < n_eff) {
        const int off = offs[si];
        uint64_t canon;
        const uint32_t f = seed_key(a, R, off, canon);
        uint4 rec = make_uint4(f, 0, 0, static_cast<uint32_t>(off));
        if (!(f & kSeedN)) {
            unsigned p = 0, m = 0;
            const bool found = probe_slot(a.table, a.n_slots, canon, p, m);
            rec = seed_record(a, f, found, p, m, off, len);
        }
        recs[lane] = rec;
    }
    __syncwarp();
}

SA_DEV void cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc) : "memory");
}
SA_DEV void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Pipelined wave 0 of the NEXT read: keys now, home slots fetched by cp.async
// into shared memory while the current read runs; resolve_wave0 finishes.
SA_DEV void issue_wave0(const AlignLaunch& a, const uint4* R, const int* offs, int n_eff,
                        uint4* recs, uint4* pslot, unsigned long long* pcanon, int lane) {
    if (lane < n_eff) {
        const int off = offs[lane];
        uint64_t canon;
        const uint32_t f = seed_key(a, R, off, canon);
        recs[lane] = make_uint4(f, 0, 0, static_cast<uint32_t>(off));
        pcanon[lane] = canon;
        if (!(f & kSeedN)) cp_async16(pslot + lane, a.table + home_slot(canon, a.n_slots));
    }
    cp_async_commit();
}

SA_DEV void resolve_wave0(const AlignLaunch& a, int n_eff, int len, uint4* recs, const uint4* pslot,
                          const unsigned long long* pcanon, int lane) {
    cp_async_wait0();
    if (lane < n_eff) {
        const uint4 rec = recs[lane];
        if (!(rec.x & kSeedN)) {
            const uint64_t canon = pcanon[lane];
            const uint4 v = pslot[lane];
            const uint64_t k = (static_cast<uint64_t>(v.y) << 32) | v.x;
            unsigned p = 0, m = 0;
            bool found;
            if (k == canon) {
                found = true;
                p = v.z;
                m = v.w;
            } else if (k == kEmptyKey) {
                found = false;
            } else {
                uint64_t h = home_slot(canon, a.n_slots) + 1;
                if (h == a.n_slots) h = 0;
                found = probe_from(a.table, a.n_slots, canon, h, p, m);
            }
            recs[lane] = seed_record(a, rec.x, found, p, m, static_cast<int>(rec.w), len);
        }
    }
    __syncwarp();
}

// Classification and result (REF aligner.cpp:318-363) and the read's
// counters, once the seed and pruning loops are over.
SA_DEV void finish_read(Ctx& x, uint32_t r, bool early_multi, bool any_popular, bool any_lookup,
                        unsigned long long& acc) {
    const AlignLaunch& a = *x.a;
    const int lane = x.lane;
    const int len = x.len;
    // classification, REF :318-363
    int kind;
    bool all_pop = false;
    const int d_max = x.d_max;
    if (early_multi) {
        kind = SA_MULTIPLE_HITS;
    } else {
        if (x.tr.d_best <= d_max && x.tr.d_second >= x.tr.d_best + a.c) kind = SA_SINGLE_HIT;
        else if (x.tr.d_best <= d_max) kind = SA_MULTIPLE_HITS;
        else kind = SA_NOT_FOUND;
        if (kind == SA_NOT_FOUND && any_popular && !any_lookup) {
            all_pop = true;
            kind = SA_MULTIPLE_HITS;
        }
    }
    sa_result res;
    res.position = 0;
    res.distance = -1;
    res.gap = 0;
    res.kind = static_cast<uint8_t>(kind);
    res.has_position = 0;
    res.direction = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i) res.reserved[i] = 0;
    bool first_best = false;
    if (kind == SA_SINGLE_HIT ||
        (kind == SA_MULTIPLE_HITS && x.tr.d_best < kInfDistance && x.tr.d_best <= d_max)) {
        res.has_position = 1;
        res.position = x.tr.best_pos;
        res.direction = static_cast<uint8_t>(x.tr.best_dir);
        res.distance = x.tr.d_best;
        res.gap = tracker_gap(x.tr);
    }
    if (kind == SA_SINGLE_HIT && x.first_valid && x.first_dir == x.tr.best_dir) {
        const uint64_t delta = x.first_pos > x.tr.best_pos ? x.first_pos - x.tr.best_pos
                                                           : x.tr.best_pos - x.first_pos;
        first_best = delta <= static_cast<uint64_t>(a.bs);
    }
    {  // sa_result as three 8-byte words, one lane each
        uint64_t w = 0;
        if (lane == 0) w = res.position;
        else if (lane == 1)
            w = static_cast<uint32_t>(res.distance) | (static_cast<uint64_t>(static_cast<uint32_t>(res.gap)) << 32);
        else if (lane == 2)
            w = res.kind | (static_cast<uint64_t>(res.has_position) << 8) | (static_cast<uint64_t>(res.direction) << 16);
        if (lane < 3) reinterpret_cast<uint64_t*>(a.results + r)[lane] = w;
    }
    stat_add(x, S_READS, 1u);
    stat_add(x, S_ALL_POP, all_pop ? 1u : 0u);
    stat_add(x, S_FIRST_BEST, first_best ? 1u : 0u);
    stat_add(x, S_SINGLE + (kind - SA_SINGLE_HIT), 1u);
    stat_add(x, S_READ_BASES, static_cast<uint32_t>(len));
    acc += x.rs;
}

// ------------------------------------------------------------------ pruning hand-off
// With a prune queue (AlignLaunch::pq_*), a read that enters the pruning loop
// (REF aligner.cpp:296-315) under a batchable bound is not pruned by the warp
// kernel: its state -- candidate table, tracker, first-scored locus, call
// count, flags and the counters so far -- goes to a record in the queue, and
// prune_kernel finishes it (prune_all, then finish_read).  The warp kernel's
// hot code then holds only the seed loop, and the pruning code runs in a
// kernel of its own.  Record layout (16-byte units from the pool base):
//   u32 r, len; i32 d_best, d_second; u64 best_pos, first_pos;
//   u32 calls, n_cands, n_unscored, flags; i32 d_max, B; u32 pad[4];
//   u32 rs[20] (lane-distributed counters); then u64 keys[n], u64 masks[n], u32 cnts[n]
constexpr uint32_t kPqHeader = 160;
enum { PQ_ANY_POP = 1, PQ_ANY_LOOKUP = 2, PQ_FIRST_DONE = 4, PQ_FIRST_VALID = 8, PQ_FIRST_DIR = 16, PQ_BEST_DIR = 32 };

SA_DEV uint32_t pq_bytes(uint32_t n) { return (kPqHeader + 20u * n + 15u) & ~15u; }

// Returns false when the pool is full (the caller prunes inline).
SA_DEV bool pq_defer(Ctx& x, uint32_t r, int B, bool any_popular, bool any_lookup) {
    const AlignLaunch& a = *x.a;
    const int lane = x.lane;
    const uint32_t n = x.n_cands;
    unsigned long long off = 0;
    if (lane == 0) off = atomicAdd(a.pq_cursor, static_cast<unsigned long long>(pq_bytes(n)));
    off = __shfl_sync(FULL, off, 0);
    if (off + pq_bytes(n) > a.pq_cap) return false;
    unsigned char* rec = a.pq_pool + off;
    if (lane == 0) {
        uint32_t* h = reinterpret_cast<uint32_t*>(rec);
        h[0] = r;
        h[1] = static_cast<uint32_t>(x.len);
        h[2] = static_cast<uint32_t>(x.tr.d_best);
        h[3] = static_cast<uint32_t>(x.tr.d_second);
        reinterpret_cast<uint64_t*>(rec)[2] = x.tr.best_pos;
        reinterpret_cast<uint64_t*>(rec)[3] = x.first_pos;
        h[8] = x.calls;
        h[9] = n;
        h[10] = x.n_unscored;
        h[11] = (any_popular ? PQ_ANY_POP : 0) | (any_lookup ? PQ_ANY_LOOKUP : 0) | (x.first_done ? PQ_FIRST_DONE : 0) |
                (x.first_valid ? PQ_FIRST_VALID : 0) | (x.first_dir ? PQ_FIRST_DIR : 0) |
                (x.tr.best_dir ? PQ_BEST_DIR : 0);
        h[12] = static_cast<uint32_t>(x.d_max);
        h[13] = static_cast<uint32_t>(B);
    }
    if (lane < kNumStats) reinterpret_cast<uint32_t*>(rec + 64)[lane] = x.rs;
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(rec + kPqHeader);
    for (uint32_t j = lane; j < n; j += 32) {
        keys[j] = x.t.ckey[j];
        keys[n + j] = x.t.cmask[j];
        reinterpret_cast<uint32_t*>(keys + 2 * n)[j] = x.t.ccnt[j];
    }
    __syncwarp();
    if (lane == 0) {
        __threadfence();
        const unsigned slot = atomicAdd(a.pq_count, 1u);
        a.pq_list[slot] = static_cast<uint32_t>(off >> 4);
    }
    return true;
}

// Align one read whose planes are already in x.R / x.C.  recs holds the seed
// records of wave 0 when wave0_ready.  Returns 0 when the candidate table
// overflowed (nothing committed), 1 when the read is done, 2 when it went to
// the prune queue.
template <bool kRegLV, bool kSlow = false, bool kSys = false>
SA_DEV int align_one(Ctx& x, uint32_t r, int n_eff, const int* offs, int tier0,
                      unsigned long long& acc, uint4* recs, bool wave0_ready, const uint4* grecs = nullptr,
                      unsigned char* pb = nullptr) {
    const AlignLaunch& a = *x.a;
    const int lane = x.lane;
    const int len = x.len;
    const bool bs_pow2 = a.bs_shift >= 0;
    const int bs_shift = a.bs_shift;

    x.n_cands = 0;
    x.n_unscored = 0;
    x.tr.d_best = kInfDistance;
    x.tr.d_second = kInfDistance;
    x.tr.best_pos = 0;
    x.tr.best_dir = 0;
    x.calls = 0;
    x.first_done = false;
    x.first_valid = false;
    x.first_dir = 0;
    x.first_pos = 0;
    x.rs = 0;
    int tested = 0;
    bool any_lookup = false, any_popular = false, early_multi = false, overflow = false;

    bool big_init = false, big_ok = false;  // kSlow: sorted pruning order
    uint32_t big_pos = 0;
    // The seed loop (REF :256-316) with the pruning loop (REF :296-315) folded
    // in, so score_best -- and the LV under it -- is inlined once.
    bool pruning = false;
    int i = 0;
    for (;;) {
        if (!pruning) {
            if (i >= n_eff) break;
            if ((i & 31) == 0 && (i > 0 || !wave0_ready)) {  // speculative probes, seeds i .. i+31
                if (grecs) {  // resolved by the seed kernel
                    __syncwarp();
                    if (i + lane < n_eff) recs[lane] = grecs[i + lane];  // resolved (resolve_kernel)
                    __syncwarp();
                } else {
                    compute_wave_sync(a, x.R, offs, i, n_eff, len, recs, lane);
                }
            }
            bool try_ff = x.n_unscored == 0;
            if (try_ff && x.n_cands == 0) {  // with no candidate yet, a seed with usable hits stops the run at once
                const uint4 r0 = recs[i & 31];
                try_ff = (r0.x & kSeedN) || r0.y == 0u || r0.y > static_cast<uint32_t>(a.hmax);
            }
            if (try_ff) {
                // Fast-forward over a run of seeds that cannot change the
                // candidate choice: N seeds, popular seeds, and lookups whose
                // hits (none, or one) land in existing candidates -- all
                // scored, as nothing is unscored.  Such a seed only moves
                // counters, and score_best / the multi exit are no-ops for it;
                // the pruning exit fires at the lookup where `tested` reaches
                // d_best + c.  Exactly the sequential loop's effect, evaluated
                // for the whole wave at once.
                const int wb = i & ~31;
                const int j = wb + lane;
                const bool in = j >= i && j < n_eff && j < wb + 32;
                const uint4 rr = recs[lane];
                const bool isN = in && (rr.x & kSeedN);
                const bool isPop = in && !isN && rr.y > static_cast<uint32_t>(a.hmax);
                const bool lk = in && !isN && !isPop;
                bool triv = lk && rr.y == 0u;
                if (lk && rr.y == 1u) {  // a single (non-palindromic) hit
                    const uint32_t dir = ((rr.x & kSeedSingleRc) ? 1u : 0u) ^ ((rr.x & kSeedQflip) ? 1u : 0u);
                    const int o = static_cast<int>(rr.w);
                    const int64_t anchor = static_cast<int64_t>(rr.z) - (dir ? (len - a.s - o) : o);
                    const uint32_t aa = anchor < 0 ? 0u : static_cast<uint32_t>(anchor);
                    const uint32_t bucket = bs_pow2 ? (aa >> bs_shift) : aa / static_cast<uint32_t>(a.bs);
                    const unsigned long long key = (static_cast<unsigned long long>(bucket) << 1) | dir;
                    for (uint32_t h = cand_hash(key, x.t.hcap);; h = (h + 1) & static_cast<uint32_t>(x.t.hcap - 1)) {
                        const unsigned long long cur = x.t.hkey[h];
                        if (cur == key) {
                            triv = true;
                            break;
                        }
                        if (cur == kEmptyKey) break;
                    }
                }
                const uint32_t m_in = __ballot_sync(FULL, in);
                const uint32_t m_n = __ballot_sync(FULL, isN);
                const uint32_t m_p = __ballot_sync(FULL, isPop);
                const uint32_t m_t = __ballot_sync(FULL, triv);
                const uint32_t m_1 = __ballot_sync(FULL, triv && rr.y == 1u);
                const uint32_t stop = m_in & ~(m_n | m_p | m_t);  // first seed needing the full path
                uint32_t run = m_in & (stop ? ((stop & (0u - stop)) - 1u) : ~0u);
                if (run != 0u) {
                    const int t0 = tier0 - wb;
                    const uint32_t below = t0 >= 32 ? ~0u : (t0 <= 0 ? 0u : ((1u << t0) - 1u));
                    const uint32_t inc = run & m_t & below;
                    const int need = x.tr.d_best + a.c - tested;  // > 0 here
                    bool prune = false;
                    if (__popc(inc) >= need) {  // exit at the need-th increment
                        uint32_t m = inc;
                        for (int k = 1; k < need; ++k) m &= m - 1u;
                        run &= (m & (0u - m)) | ((m & (0u - m)) - 1u);
                        prune = true;
                    }
                    stat_add(x, S_SKIP_N, __popc(run & m_n));
                    stat_add(x, S_LOOKUPS, __popc(run & ~m_n));
                    stat_add(x, S_SKIP_POP, __popc(run & m_p));
                    stat_add(x, S_HITS, __popc(run & m_1));
                    tested += __popc(run & inc);
                    any_popular |= (run & m_p) != 0u;
                    any_lookup |= (run & m_t) != 0u;
                    if (prune) {  // REF :296-315 with nothing unscored
                        stat_add(x, S_PRUNE, 1u);
                        break;
                    }
                    i = wb + 32 - __clz(run);  // one past the run's last seed
                    continue;
                }
            }
            const uint4 rec = recs[i & 31];
            const uint32_t flags = rec.x;
            const uint32_t cnt = rec.y;
            if (flags & kSeedN) {  // REF :259-262
                stat_add(x, S_SKIP_N, 1u);
                ++i;
                continue;
            }
            stat_add(x, S_LOOKUPS, 1u);
            if (cnt > static_cast<uint32_t>(a.hmax)) {  // REF :265-269
                any_popular = true;
                stat_add(x, S_SKIP_POP, 1u);
                ++i;
                continue;
            }
            any_lookup = true;
            stat_add(x, S_HITS, cnt);
            if (i < tier0) ++tested;

            if (cnt > 0) {  // REF :273-286
                const uint32_t payload = rec.z;
                const int off = static_cast<int>(rec.w);
                const bool pal = (flags & kSeedPal) != 0;
                const uint32_t ntot = pal ? cnt / 2 : cnt;
                const bool inl = ntot == 1;
                uint32_t n_fwd = 0;
                if (!inl) n_fwd = __ldg(a.pool + payload);
                const int rc_shift = len - a.s - off;
                const uint32_t qflip = (flags & kSeedQflip) ? 1u : 0u;
                for (uint32_t base = 0; base < cnt; base += 32) {
                    const uint32_t t = base + lane;
                    const bool valid = t < cnt;
                    unsigned long long key = 0;
                    int bit = 0;
                    if (valid) {
                        const uint32_t j = pal ? (t < ntot ? t : t - ntot) : t;
                        uint32_t pos, eflag;
                        if (inl) {
                            pos = payload;
                            eflag = (flags & kSeedSingleRc) ? 1u : 0u;
                        } else {
                            pos = __ldg(a.pool + payload + 1 + j);
                            eflag = j >= n_fwd ? 1u : 0u;
                        }
                        const uint32_t dir = pal ? (t >= ntot ? 1u : 0u) : (eflag ^ qflip);
                        const int64_t anchor = static_cast<int64_t>(pos) - (dir ? rc_shift : off);
                        const uint32_t aa = anchor < 0 ? 0u : static_cast<uint32_t>(anchor);
                        uint32_t bucket;
                        if (bs_pow2) {
                            bucket = aa >> bs_shift;
                            bit = static_cast<int>(aa & static_cast<uint32_t>(a.bs - 1));
                        } else {
                            bucket = aa / static_cast<uint32_t>(a.bs);
                            bit = static_cast<int>(aa - bucket * static_cast<uint32_t>(a.bs));
                        }
                        key = (static_cast<unsigned long long>(bucket) << 1) | dir;
                    }
                    if (!insert_wave(x, valid, key, bit)) {
                        overflow = true;
                        break;
                    }
                }
                if (overflow) break;
            }

        } else if (x.n_unscored == 0) {
            break;
        }
#if SA_PRUNE_BATCH
        // the batch exists only for short-read layouts (d_limit <= 15: the
        // register-LV kernels); the long-read kernels are compiled without it
        if (kRegLV && pruning && pb != nullptr) {  // the rest of the pruning loop, a batch at a time
            const int cmax = x.d_max + a.c - 1;
            const int B = (a.force || x.tr.d_best > x.d_max) ? cmax : x.tr.d_best + a.c - 1;
            if (B >= 0 && B <= kPbMax) {
                if (a.pq_pool) {  // to prune_kernel; a full pool sends the read to the global-table pass
                    const bool ok = pq_defer(x, r, B, any_popular, any_lookup);
                    clear_table(x.t, x.n_cands, !ok, lane);
                    return ok ? 2 : 0;
                }
#if SA_DEBUG_COUNTERS
                if (a.dbg && lane == 0) {  // pruning batches: entries, candidates, B sum
                    atomicAdd(a.dbg + 7, 1u);
                    atomicAdd(a.dbg + 8, x.n_unscored);
                    atomicAdd(a.dbg + 9, static_cast<unsigned>(B));
                }
#endif
                if (prune_all(x, pb, B)) {
                    stat_add(x, S_MULTI, 1u);
                    early_multi = true;
                }
                break;
            }
        }
#endif
        if (kSlow && pruning) {
            // global-table kernel, pruning loop without the batch (long reads):
            // the loop's order sorted once (select_order_large), then scored
            // candidate by candidate, instead of an argmax over the table each time
            if (!big_init) {
                big_init = true;
                big_ok = x.n_cands > 64 && x.t.hcap >= 2 * x.t.cap &&
                         select_order_large(x, reinterpret_cast<unsigned long long*>(x.t.hval));
                big_pos = 0;
            }
            if (big_ok) {
                const unsigned long long* big = reinterpret_cast<const unsigned long long*>(x.t.hval);
                score_candidate<kRegLV, kSys>(x, static_cast<uint32_t>(big[big_pos++] & 0x3fffu));
            } else {
                score_best<kRegLV, kSys>(x);
            }
        } else {
            score_best<kRegLV, kSys>(x);  // REF :288 (and :306 inside the pruning loop)
        }
        if (x.tr.d_best < a.c && x.tr.d_second < x.tr.d_best + a.c) {  // REF :290-295 / :307-312
            stat_add(x, S_MULTI, 1u);
            early_multi = true;
            break;
        }
        if (!pruning) {
            if (tested >= x.tr.d_best + a.c) {  // REF :296-315
                stat_add(x, S_PRUNE, 1u);
                pruning = true;
            }
            ++i;
        }
    }

    if (overflow) {
        clear_table(x.t, x.n_cands, true, lane);
        return 0;
    }
    clear_table(x.t, x.n_cands, false, lane);
    finish_read(x, r, early_multi, any_popular, any_lookup, acc);
    return 1;
}

// ------------------------------------------------------------------ solo kernel
// Thread-per-read aligner for the common read (two-kernel path, register-LV
// launches, power-of-two bucket <= 32).  The warp-per-read kernel spends most
// of its ~1,300 warp-instructions per read on control flow that is the same
// for all 32 lanes; here one thread replays Aligner::align (REF
// src/aligner.cpp:223-364) for its own read from the seed kernel's records,
// with the candidate table and the LV frontier in its own shared-memory
// column, so all 32 lanes do useful work.  A read it cannot finish within its
// limits -- a seed with more than SA_SOLO_MAX_HITS hits (palindromes
// included), more than kSoloCands candidates, a bad character or a deferred
// length -- is appended to pre_list untouched and the warp kernel redoes it
// from scratch, so the result is the same whichever kernel finishes a read.
// The steps are align_one's (same d_limit rule, candidate order, LV steps,
// tracker, exits, classification and counters), written per lane as a state
// machine the warp walks together (seed phase, LV phase).
#ifndef SA_SOLO_CANDS
#define SA_SOLO_CANDS 8
#endif
constexpr int kSoloCands = SA_SOLO_CANDS;
#ifndef SA_SOLO_THREADS
#define SA_SOLO_THREADS 128
#endif
constexpr int kSoloThreads = SA_SOLO_THREADS;
constexpr int kSoloF = 2 * 15 + 3;  // frontier entries at d_limit <= 15

#ifndef SA_SOLO_PF
#define SA_SOLO_PF 2  // prefetch a read's records and planes at its start: 1 into L2, 2 into L1 (C1 969 -> 991 M reads/s)
#endif
SA_DEV void solo_prefetch(const void* p) {
#if SA_SOLO_PF == 2
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
#else
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
#endif
}

struct SoloRead {
    uint32_t lookups = 0, skip_n = 0, skip_pop = 0, hits = 0, dist = 0, dist_after = 0, early_out = 0;
    uint32_t window = 0, cells = 0, multi = 0, prune = 0;
};

#ifndef SA_SOLO_MIN_BLOCKS
#define SA_SOLO_MIN_BLOCKS 7  // 72 registers, 28 warps per SM (6 blocks / 80 registers: C2 497 -> 499 M, C1 1,485 -> 1,540 M reads/s; 8 blocks / 64 registers: 500 / 1,475 M)
#endif
#ifndef SA_SOLO_LV
// solo LV: 0 serial wavefront (lv_thread); 1 banded bit-parallel (lv_bitpar).
// Measured at C1: 0 -> 934 M reads/s, 1 -> 591 M (a fixed m + d_limit column
// steps per call against the wavefront's few steps for a close read), and a
// single-loop (flattened) wavefront 737 M.
#define SA_SOLO_LV 0
#endif
#ifndef SA_SOLO_MAX_HITS
#define SA_SOLO_MAX_HITS 6  // hits of one seed the thread votes itself (more: the warp kernel; C2 4/6/8 with the phase-synchronous kernel: 485/492/487 M reads/s)
#endif
#ifndef SA_SOLO_MAX_E
#define SA_SOLO_MAX_E 2  // LV iterations a thread runs serially
#endif
#ifndef SA_SOLO_COOP
#define SA_SOLO_COOP 1  // 1: the warp finishes longer wavefronts lane per diagonal; 0: their reads go to the warp kernel
#endif
__global__ void __launch_bounds__(kSoloThreads, SA_SOLO_MIN_BLOCKS) solo_kernel(const AlignLaunch a) {
    __shared__ uint32_t s_key[kSoloCands][kSoloThreads];   // bucket << 1 | dir
    __shared__ uint32_t s_mask[kSoloCands][kSoloThreads];  // anchor bits (bucket <= 32)
    __shared__ uint32_t s_cnt[kSoloCands][kSoloThreads];   // seeds_hitting | kScored
#if SA_SOLO_LV != 1
    __shared__ short s_F[kSoloF][kSoloThreads];
#endif
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    uint32_t* ckey = &s_key[0][tid];
    uint32_t* cmask = &s_mask[0][tid];
    uint32_t* ccnt = &s_cnt[0][tid];
    constexpr int cs = kSoloThreads;  // column stride
    const int half = a.pre_pstride >> 1;
    const int bsh = a.bs_shift;
    unsigned long long acc = 0;  // lane k: stats slot k of the warp
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x; base < a.n_reads; base += stride) {
        const uint32_t r = base + tid;
        // per-read outcome: 0 none, 1 committed, 2 complex (warp kernel)
        int outcome = 0;
        SoloRead c;
        int kind = SA_NOT_FOUND, len = 0;
        bool all_pop = false, first_best = false, too_short = false;
        // The read's alignment is a small state machine so the warp stays
        // converged where it matters: every lane first advances its own seed
        // loop up to its next LV job (kSeed), then all lanes holding a job run
        // their LVs together (kLv) -- entered one by one from divergent seed-loop
        // paths the LV code, 70% of this kernel's instructions, ran with 2.8
        // active lanes per instruction (profiles/r02y_ncu_C2.md).
        enum { kIdle = 0, kSeed, kLv, kClassify };
        int phase = kIdle;
        const uint4* recs = nullptr;
        const uint4* Rp = nullptr;
        int n_eff = 0, d_max = 0, tier0 = 0;
        Tracker tr;
        tr.d_best = kInfDistance;
        tr.d_second = kInfDistance;
        tr.best_pos = 0;
        tr.best_dir = 0;
        uint32_t n_cands = 0, n_unscored = 0, calls = 0;
        bool first_done = false, first_valid = false;
        int first_dir = 0;
        uint64_t first_pos = 0;
        int tested = 0;
        bool any_lookup = false, any_popular = false, early_multi = false, pruning = false;
        int i = 0;
        // the LV job: candidate key, anchors left, limit, best so far
        uint32_t job_kk = 0, job_mm = 0;
        int job_dl = 0, job_best_d = kInfDistance;
        uint64_t job_best_anchor = 0;
        if (r < a.n_reads) {
            const uint2 meta = __ldg(a.pre_meta + r);
            len = static_cast<int>(meta.x);
            const uint32_t st = meta.y >> 16;
            n_eff = static_cast<int>(meta.y & 0xffffu);
            outcome = 2;
            if (st == 1) {  // REF aligner.cpp:231-235
                sa_result res;
                res.position = 0;
                res.distance = -1;
                res.gap = 0;
                res.kind = SA_NOT_FOUND;
                res.has_position = 0;
                res.direction = 0;
#pragma unroll
                for (int q = 0; q < 5; ++q) res.reserved[q] = 0;
                a.results[r] = res;
                too_short = true;
                outcome = 1;
            } else if (st == 0) {
                recs = a.pre_recs + static_cast<uint64_t>(r) * a.pre_rstride;
                Rp = a.pre_planes + static_cast<uint64_t>(r) * a.pre_pstride;
#if SA_SOLO_PF
                // the seed loop reads the records one by one behind data-dependent
                // branches, and the LV walks the planes as the wavefront advances:
                // touch their lines up front so those loads find them close
                for (int t = 0; t < n_eff && t < 16; t += 2) solo_prefetch(recs + t);  // 2 records per 32 B sector
                for (int t = 0; t < a.pre_pstride && t < 16; t += 2) solo_prefetch(Rp + t);
#endif
                d_max = a.dmax_param >= 0 ? a.dmax_param : (12 * len + 99) / 100;
                tier0 = len / a.s;
                phase = kSeed;
            }
        }
        // after a seed's scoring step (REF :290-315): multi exit, pruning switch, next seed
        auto after_step = [&]() {
            if (tr.d_best < a.c && tr.d_second < tr.d_best + a.c) {  // REF :290-295 / :307-312
                c.multi++;
                early_multi = true;
                phase = kClassify;
                return;
            }
            if (!pruning) {
                if (tested >= tr.d_best + a.c) {  // REF :296-315
                    c.prune++;
                    pruning = true;
                }
                ++i;
            }
        };
        for (;;) {
            // ---- kSeed: this lane's seed loop up to its next LV job
            // (structured branches only -- no continue/break out of the body --
            // so the lanes rejoin after every step of the loop)
            while (phase == kSeed) {
                bool score = false;  // this step goes on to score_best_candidate
                if (pruning) {
                    if (n_unscored == 0) phase = kClassify;
                    else score = true;
                } else if (i >= n_eff) {
                    phase = kClassify;
                } else {
                    uint4 rec = __ldg(recs + i);
                    if (rec.x & kSeedLazy) rec = resolve_lazy(a, rec);  // probed on demand
                    if (rec.x & kSeedN) {  // REF :259-262
                        c.skip_n++;
                        ++i;
                    } else if (rec.y > static_cast<uint32_t>(a.hmax)) {  // REF :265-269
                        c.lookups++;
                        any_popular = true;
                        c.skip_pop++;
                        ++i;
                    } else if (rec.y > static_cast<uint32_t>(SA_SOLO_MAX_HITS)) {  // long vote lists: the warp kernel
                        if (a.dbg) atomicAdd(a.dbg + 0, 1u);
                        phase = kIdle;
                    } else {
                        c.lookups++;
                        any_lookup = true;
                        c.hits += rec.y;
                        if (i < tier0) ++tested;
                        // REF :273-286: every hit of the seed votes for (anchor / bucket, dir)
                        const uint32_t cnt = rec.y;
                        const bool pal = (rec.x & kSeedPal) != 0;
                        const uint32_t ntot = pal ? cnt / 2 : cnt;
                        const bool inl = ntot == 1;
                        const uint32_t n_fwd = inl ? 0u : __ldg(a.pool + rec.z);
                        const uint32_t qflip = (rec.x & kSeedQflip) ? 1u : 0u;
                        const int o = static_cast<int>(rec.w);
                        bool full = false;
                        for (uint32_t t = 0; t < cnt && !full; ++t) {
                            const uint32_t jj = pal ? (t < ntot ? t : t - ntot) : t;
                            uint32_t pos, eflag;
                            if (inl) {
                                pos = rec.z;
                                eflag = (rec.x & kSeedSingleRc) ? 1u : 0u;
                            } else {
                                pos = __ldg(a.pool + rec.z + 1 + jj);
                                eflag = jj >= n_fwd ? 1u : 0u;
                            }
                            const uint32_t dir = pal ? (t >= ntot ? 1u : 0u) : (eflag ^ qflip);
                            const int64_t anchor = static_cast<int64_t>(pos) - (dir ? (len - a.s - o) : o);
                            const uint32_t aa = anchor < 0 ? 0u : static_cast<uint32_t>(anchor);
                            const uint32_t key = ((aa >> bsh) << 1) | dir;
                            const uint32_t bit = 1u << (aa & ((1u << bsh) - 1u));
                            uint32_t j = 0;
                            while (j < n_cands && ckey[j * cs] != key) ++j;
                            if (j < n_cands) {
                                ccnt[j * cs] += 1u;
                                cmask[j * cs] |= bit;
                            } else if (n_cands == kSoloCands) {  // more candidates than the table holds
                                if (a.dbg) atomicAdd(a.dbg + 1, 1u);
                                full = true;
                            } else {
                                ckey[j * cs] = key;
                                cmask[j * cs] = bit;
                                ccnt[j * cs] = 1u;
                                ++n_cands;
                                ++n_unscored;
                            }
                        }
                        if (full) phase = kIdle;  // the warp kernel
                        else score = true;
                    }
                }
                if (score) {
                    bool job = false;
                    // score_best_candidate (REF :141-167)
                    if (n_unscored > 0) {
                        uint32_t bi = 0, bc = 0;
                        uint64_t bord = ~0ull;
                        for (uint32_t j = 0; j < n_cands; ++j) {
                            const uint32_t cc = ccnt[j * cs];
                            const uint32_t kk = ckey[j * cs];
                            // amin = bucket * bs + lowest bit; order (amin, dir) as (amin << 1 | dir)
                            const uint64_t amin = (static_cast<uint64_t>(kk >> 1) << bsh) + (__ffs(cmask[j * cs]) - 1);
                            const uint64_t ord = (amin << 1) | (kk & 1u);
                            if (!(cc & kScored) && (cc > bc || (cc == bc && ord < bord))) {
                                bc = cc;
                                bord = ord;
                                bi = j;
                            }
                        }
                        // score_candidate (REF :169-221): the LVs run in the kLv phase
                        ccnt[bi * cs] |= kScored;
                        --n_unscored;
                        int d_limit;
                        if (tr.d_best > d_max) d_limit = d_max + a.c - 1;
                        else if (tr.d_second >= tr.d_best + a.c) d_limit = tr.d_best + a.c - 1;
                        else d_limit = tr.d_best - 1;
                        if (a.force) d_limit = d_max + a.c - 1;
                        if (d_limit >= 0) {  // (:184)
                            job_kk = ckey[bi * cs];
                            job_mm = cmask[bi * cs];
                            job_dl = d_limit;
                            job_best_d = kInfDistance;
                            job_best_anchor = 0;
                            phase = kLv;
                            job = true;
                        }
                    }
                    if (!job) after_step();
                }
            }
            // ---- kLv: one anchor's LV per lane, all lanes with a job together
            if (!__any_sync(FULL, phase == kLv)) break;  // no lane is left in kSeed here
            const int dir = static_cast<int>(job_kk & 1u);
            bool have = false;
            uint64_t anchor = 0;
            int w = 0, d = -1;
            if (phase == kLv) {
                const uint64_t base_pos = static_cast<uint64_t>(job_kk >> 1) << bsh;
                while (job_mm != 0u && !have) {
                    anchor = base_pos + static_cast<uint64_t>(__ffs(job_mm) - 1);
                    job_mm &= job_mm - 1u;
                    have = anchor < a.glen;
                }
                if (have) {
                    const uint64_t rem = a.glen - anchor;
                    const uint64_t want = static_cast<uint64_t>(len) + static_cast<uint64_t>(job_dl);
                    w = static_cast<int>(want < rem ? want : rem);
#if SA_SOLO_LV == 1
                    d = lv_bitpar(Rp + (dir ? half : 0), half, len, a.planes, static_cast<uint32_t>(anchor), w, job_dl,
                                  c.cells);
#else
                    d = lv_thread(Rp + (dir ? half : 0), len, a.planes, static_cast<uint32_t>(anchor), w, job_dl,
                                  &s_F[0][tid], cs, c.cells, SA_SOLO_MAX_E);
#endif
                }
            }
#if SA_SOLO_COOP && SA_SOLO_LV != 1
            // The wavefronts still open after SA_SOLO_MAX_E serial iterations are
            // few and wide (2e + 1 diagonals each): the warp finishes them one at a
            // time, lane per diagonal, from the owner's frontier column.
            __syncwarp();  // the owners' frontier columns are read by the other lanes
            for (uint32_t pend = __ballot_sync(FULL, d == -2); pend != 0u; pend &= pend - 1u) {
                const int src = __ffs(pend) - 1;
                const uint4* Rb = reinterpret_cast<const uint4*>(
                    shfl64(reinterpret_cast<unsigned long long>(Rp + (dir ? half : 0)), src));
                const uint32_t wofs = __shfl_sync(FULL, static_cast<uint32_t>(anchor), src);
                const int wb = __shfl_sync(FULL, w, src), dlb = __shfl_sync(FULL, job_dl, src);
                const int mb = __shfl_sync(FULL, len, src);
                uint32_t cells = 0;  // every lane's steps count for the owner's read
                const int res = lv_warp_resume(Rb, mb, a.planes, wofs, wb, dlb, &s_F[0][(tid & ~31) + src], cs,
                                               SA_SOLO_MAX_E, lane, cells);
                cells = __reduce_add_sync(FULL, cells);
                if (lane == src) {
                    d = res;
                    c.cells += cells;
                }
            }
#endif
            if (phase == kLv) {
                if (d == -2) {  // a long wavefront: the warp kernel
                    if (a.dbg) atomicAdd(a.dbg + 2, 1u);
                    phase = kIdle;
                } else {
                    if (have) {
                        c.dist++;
                        calls++;
                        c.window += static_cast<uint32_t>(w);
                        if (calls > 1) {
                            c.dist_after++;
                            if (d < 0) c.early_out++;
                        }
                        if (d >= 0 && d < job_best_d) {
                            job_best_d = d;
                            job_best_anchor = anchor;
                        }
                    }
                    if (job_mm == 0u) {  // the candidate's anchors are done
                        if (!first_done) {
                            first_done = true;
                            if (job_best_d < kInfDistance) {
                                first_valid = true;
                                first_pos = job_best_anchor;
                                first_dir = dir;
                            }
                        }
                        if (job_best_d < kInfDistance) tracker_observe(tr, a.bs, job_best_d, job_best_anchor, dir);
                        phase = kSeed;
                        after_step();
                    }
                }
            }
        }
        if (phase == kClassify) {  // classification, REF :318-363
            if (early_multi) {
                kind = SA_MULTIPLE_HITS;
            } else {
                if (tr.d_best <= d_max && tr.d_second >= tr.d_best + a.c) kind = SA_SINGLE_HIT;
                else if (tr.d_best <= d_max) kind = SA_MULTIPLE_HITS;
                else kind = SA_NOT_FOUND;
                if (kind == SA_NOT_FOUND && any_popular && !any_lookup) {
                    all_pop = true;
                    kind = SA_MULTIPLE_HITS;
                }
            }
            uint64_t w0 = 0, w1 = static_cast<uint32_t>(-1), w2 = static_cast<uint64_t>(kind);
            if (kind == SA_SINGLE_HIT || (kind == SA_MULTIPLE_HITS && tr.d_best <= d_max)) {
                w0 = tr.best_pos;
                w1 = static_cast<uint32_t>(tr.d_best) |
                     (static_cast<uint64_t>(static_cast<uint32_t>(tracker_gap(tr))) << 32);
                w2 |= (1ull << 8) | (static_cast<uint64_t>(tr.best_dir) << 16);
            }
            if (kind == SA_SINGLE_HIT && first_valid && first_dir == tr.best_dir) {
                const uint64_t delta = first_pos > tr.best_pos ? first_pos - tr.best_pos : tr.best_pos - first_pos;
                first_best = delta <= static_cast<uint64_t>(a.bs);
            }
            uint64_t* out = reinterpret_cast<uint64_t*>(a.results + r);
            out[0] = w0;
            out[1] = w1;
            out[2] = w2;
            outcome = 1;
        }
        // reads for the warp kernel, warp-aggregated
        const uint32_t cm = __ballot_sync(FULL, outcome == 2);
        if (cm) {
            unsigned int slot0 = 0;
            if (lane == __ffs(cm) - 1) slot0 = atomicAdd(a.pre_list_count, static_cast<unsigned>(__popc(cm)));
            slot0 = __shfl_sync(FULL, slot0, __ffs(cm) - 1);
            if (outcome == 2) a.pre_list[slot0 + __popc(cm & lanemask_lt())] = r;
        }
        if (__any_sync(FULL, outcome == 1)) {  // counters of the committed reads, one slot per lane
            const bool ok = outcome == 1;
            const bool full = ok && !too_short;
            auto put = [&](int slot, uint32_t v) {
                const uint32_t t = __reduce_add_sync(FULL, v);
                if (lane == slot) acc += t;
            };
            put(S_READS, ok ? 1u : 0u);
            put(S_TOO_SHORT, too_short ? 1u : 0u);
            put(S_READ_BASES, ok ? static_cast<uint32_t>(len) : 0u);
            put(S_SINGLE, full && kind == SA_SINGLE_HIT ? 1u : 0u);
            put(S_MULTIPLE, full && kind == SA_MULTIPLE_HITS ? 1u : 0u);
            put(S_NOT_FOUND, ok && kind == SA_NOT_FOUND ? 1u : 0u);
            put(S_ALL_POP, full && all_pop ? 1u : 0u);
            put(S_FIRST_BEST, full && first_best ? 1u : 0u);
            put(S_LOOKUPS, full ? c.lookups : 0u);
            put(S_SKIP_N, full ? c.skip_n : 0u);
            put(S_SKIP_POP, full ? c.skip_pop : 0u);
            put(S_HITS, full ? c.hits : 0u);
            put(S_DIST, full ? c.dist : 0u);
            put(S_DIST_AFTER, full ? c.dist_after : 0u);
            put(S_EARLY_OUT, full ? c.early_out : 0u);
            put(S_WINDOW, full ? c.window : 0u);
            put(S_CELLS, full ? c.cells : 0u);
            put(S_MULTI, full ? c.multi : 0u);
            put(S_PRUNE, full ? c.prune : 0u);
        }
    }
    if (lane < kNumStats && acc) atomicAdd(a.stats + lane, acc);
}

// The reads solo_kernel listed for the warp kernel still hold the lazy
// records it did not reach: one thread per (listed read, seed) probes them
// here, all at once, instead of each warp kernel read paying a dependent
// round of probes when it starts.
__global__ void __launch_bounds__(256) resolve_kernel(const AlignLaunch a) {
    const uint32_t n = *a.pre_list_count;
    const uint32_t nr = static_cast<uint32_t>(a.pre_rstride);
    const uint64_t total = static_cast<uint64_t>(n) * nr;
    for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t r = __ldg(a.pre_list + t / nr);
        const uint32_t sd = static_cast<uint32_t>(t % nr);
        const uint2 meta = __ldg(a.pre_meta + r);
        if ((meta.y >> 16) != 0 || sd >= (meta.y & 0xffffu)) continue;
        uint4* rec = a.pre_recs + static_cast<uint64_t>(r) * a.pre_rstride + sd;
        const uint4 v = *rec;
        if (v.x & kSeedLazy) *rec = resolve_lazy(a, v);
    }
}

// ------------------------------------------------------------------ seed kernel
// Stage 1 of the two-kernel path: one thread per read (full lane use, and
// the probes of a whole warp of reads in flight at once).  Decodes the read
// into forward and reverse-complement planes (REF genome.cpp:182-200), lists
// its seed offsets (REF aligner.cpp:50-79) and resolves every seed against
// the index (REF seed_index.cpp:128-143) into the same records the align
// kernel's waves use.
// A group of G lanes (G = power of two >= the launch's blocks per read, at
// most 32) handles one read: lane g decodes 32-base block g with coalesced
// word loads and SWAR compares, the reverse-complement blocks and the seed
// windows are assembled with shuffles inside the group, and the read's seeds
// are dealt round-robin to the lanes so their index probes are in flight
// together.
// seed_offsets (REF aligner.cpp:50-79) for one length, sequentially: the
// tier-0 non-overlapping offsets 0, s, 2s, ... first, then the same ladder
// from each shift (odd * s) >> level of successive binary subdivisions of
// [0, s), skipping shifts already used, until n_cap offsets or the shifts run
// out -- the generator the seed kernel's lanes walk (next_off below).
constexpr int kSeedTab = 64;
SA_DEV int seed_offsets_list(int len, int s, int n_cap, int* out) {
    const int max_off = len - s;
    uint32_t used = 1u;  // shift 0: the tier-0 ladder
    int cnt = 0;
    for (int o = 0; o <= max_off && cnt < n_cap; o += s) out[cnt++] = o;
    for (int level = 1, odd = 1; cnt < n_cap;) {
        if ((1 << level) > 4 * s) break;
        const int shift = (odd * s) >> level;
        odd += 2;
        if (odd >= (1 << level)) {
            ++level;
            odd = 1;
        }
        if ((used >> shift) & 1u) continue;
        used |= 1u << shift;
        for (int o = shift; o <= max_off && cnt < n_cap; o += s) out[cnt++] = o;
    }
    return cnt;
}

#ifndef SA_SEED_MIN_BLOCKS
#define SA_SEED_MIN_BLOCKS 6  // 40 registers: 48 warps per SM (measured +2.5% over the unbounded 42-register build)
#endif
template <int G>
__global__ void __launch_bounds__(256, SA_SEED_MIN_BLOCKS) seed_kernel(const AlignLaunch a) {
    const int lane = threadIdx.x & 31;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (a.pre_list_count) *a.pre_list_count = 0;  // solo_kernel appends next
        if (a.work_cursor) *a.work_cursor = 0;         // the warp kernel's read cursor
        if (a.pq_cursor) {                             // the warp kernel's prune queue
            *a.pq_cursor = 0;
            *a.pq_count = 0;
            *a.pq_cursor2 = 0;
        }
    }
    const int g = lane & (G - 1);
    const int gbase = lane & ~(G - 1);
    const uint32_t groups = (gridDim.x * blockDim.x) / G;
    const int half = a.pre_pstride >> 1;
    // The seed offsets (REF aligner.cpp:50-79) depend only on the read length:
    // the block lists them once for the length of its first read, and every
    // read of that length takes them from shared memory instead of walking the
    // generator in each lane (a quarter of this kernel's instructions).
    __shared__ int s_off[kSeedTab];
    __shared__ int s_tab_len, s_tab_n;
    if (threadIdx.x == 0) {
        s_tab_len = -1;
        const uint32_t r0 = (blockIdx.x * blockDim.x) / G;
        const int n_cap = min(a.n, a.n_off_cap);
        if (r0 < a.n_reads && n_cap <= kSeedTab) {
            const int len0 = a.fixed_len ? static_cast<int>(a.fixed_len)
                                         : static_cast<int>(a.offsets[r0 + 1] - a.offsets[r0]);
            if (len0 >= a.s && len0 <= a.lcap) {
                s_tab_n = seed_offsets_list(len0, a.s, n_cap, s_off);
                s_tab_len = len0;
            }
        }
    }
    __syncthreads();
    const int tab_len = s_tab_len, tab_n = s_tab_n;
    const uint32_t gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << gbase);
    // all groups of a warp iterate the same number of times (shuffles)
    const uint32_t first = (blockIdx.x * blockDim.x + threadIdx.x) / G;
    const uint32_t n_iter = (a.n_reads + groups - 1) / groups;
    for (uint32_t it = 0; it < n_iter; ++it) {
        const uint32_t r = first + it * groups;
        const bool live = r < a.n_reads;
        int len = 0;
        uint64_t o0 = 0;
        if (live) {
            if (a.fixed_len) {
                o0 = a.base_off + static_cast<uint64_t>(r) * a.fixed_len;
                len = static_cast<int>(a.fixed_len);
            } else {
                o0 = a.offsets[r];
                len = static_cast<int>(a.offsets[r + 1] - o0);
            }
        }
        uint32_t status = 0;
        if (!live) status = 4;
        else if (len < a.s) status = 1;
        else if (len > a.lcap) status = 3;
        const int nb = (len + 31) >> 5;
        // ---- decode block g (REF genome.cpp:182-200 alphabet)
        uint32_t lo = 0, hi = 0, nn = 0xffffffffu, bad = 0;
        if (a.packed != nullptr) {  // host-packed planes (pack.cpp)
            if (status == 0 && g < nb) {
                const uint64_t p = (o0 - a.base_off) + 32ull * static_cast<uint64_t>(g);
                const uint32_t* P0 = a.packed + (p >> 5);
                const uint32_t sh = static_cast<uint32_t>(p & 31);
                lo = __funnelshift_r(__ldg(P0), __ldg(P0 + 1), sh);
                hi = __funnelshift_r(__ldg(P0 + a.pk_wpp), __ldg(P0 + a.pk_wpp + 1), sh);
                nn = __funnelshift_r(__ldg(P0 + 2 * a.pk_wpp), __ldg(P0 + 2 * a.pk_wpp + 1), sh);
                const int avail = len - 32 * g;
                if (avail < 32) {  // beyond the read: N
                    const uint32_t keep = (1u << avail) - 1u;
                    lo &= keep;
                    hi &= keep;
                    nn = (nn & keep) | ~keep;
                }
                bad = lo & nn;
            }
        } else if (status == 0 && g < nb) {
            const uintptr_t addr = reinterpret_cast<uintptr_t>(a.bases + (o0 - a.base_off)) + 32u * g;
            const uint32_t* W = reinterpret_cast<const uint32_t*>(addr & ~static_cast<uintptr_t>(3));
            const uint32_t sh = 8u * static_cast<uint32_t>(addr & 3);
            const int avail = len - 32 * g;  // bases of this block present
            const uint32_t* Wend = reinterpret_cast<const uint32_t*>(
                (reinterpret_cast<uintptr_t>(a.bases + (o0 - a.base_off)) + len + 3) & ~static_cast<uintptr_t>(3));
            nn = 0;
            uint32_t w0 = __ldg(W);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                uint32_t v = 0x4E4E4E4Eu;
                if (4 * k < avail) {
                    const uint32_t w1 = (W + k + 1 < Wend) ? __ldg(W + k + 1) : 0u;
                    v = __funnelshift_r(w0, w1, sh);
                    w0 = w1;
                    const int valid = avail - 4 * k;
                    if (valid < 4) {
                        const uint32_t keep = (1u << (8 * valid)) - 1u;
                        v = (v & keep) | (0x4E4E4E4Eu & ~keep);
                    }
                }
                uint32_t l4, h4, n4, b4;
                decode4(v, l4, h4, n4, b4);
                bad |= b4;
                lo |= l4 << (4 * k);
                hi |= h4 << (4 * k);
                nn |= n4 << (4 * k);
            }
        }
        const bool any_bad = (__ballot_sync(gmask, bad != 0) & gmask) != 0;
        if (status == 0 && any_bad) status = 2;
        // 32 forward bases starting at base p (< len), from the group's blocks
        auto fwd32 = [&](int pq, uint32_t& l, uint32_t& h, uint32_t& n) {
            const int b = pq >> 5, sft = pq & 31;
            const int src0 = gbase + (b < G ? b : G - 1), src1 = gbase + (b + 1 < G ? b + 1 : G - 1);
            const uint32_t l0 = __shfl_sync(gmask, lo, src0), l1 = __shfl_sync(gmask, lo, src1);
            const uint32_t h0 = __shfl_sync(gmask, hi, src0), h1 = __shfl_sync(gmask, hi, src1);
            const uint32_t n0 = __shfl_sync(gmask, nn, src0), n1 = __shfl_sync(gmask, nn, src1);
            const bool in1 = b + 1 < nb;  // beyond the read: N
            l = __funnelshift_r(l0, in1 ? l1 : 0u, sft);
            h = __funnelshift_r(h0, in1 ? h1 : 0u, sft);
            n = __funnelshift_r(n0, in1 ? n1 : 0xffffffffu, sft);
        };
        // ---- reverse complement block g: bit b = complement of base len-1-32g-b
        uint32_t rl = 0, rh = 0, rn = 0xffffffffu;
        {
            const int p_lo = len - 32 * (g + 1);
            uint32_t l, h, n;
            fwd32(p_lo >= 0 ? p_lo : 0, l, h, n);
            if (p_lo < 0) {
                const int sft = -p_lo;
                l = sft >= 32 ? 0u : l << sft;
                h = sft >= 32 ? 0u : h << sft;
                n = sft >= 32 ? 0xffffffffu : ((n << sft) | ((1u << sft) - 1u));
            }
            if (status == 0 && g < nb) {
                rl = __brev(~l);
                rh = __brev(~h);
                rn = __brev(n);
            }
        }
        if (status == 0) {
            uint4* P = a.pre_planes + static_cast<uint64_t>(r) * a.pre_pstride;
            if (g <= nb && g < half) {
                P[g] = g < nb ? make_uint4(lo, hi, nn, 0) : make_uint4(0, 0, 0xFFFFFFFFu, 0);
                P[half + g] = g < nb ? make_uint4(rl, rh, rn, 0) : make_uint4(0, 0, 0xFFFFFFFFu, 0);
            }
            if (g == 0 && nb == G && nb < half) {  // the all-N pad block has no lane of its own
                P[nb] = make_uint4(0, 0, 0xFFFFFFFFu, 0);
                P[half + nb] = make_uint4(0, 0, 0xFFFFFFFFu, 0);
            }
        }
        // ---- seeds: offsets (REF aligner.cpp:50-79) dealt round-robin; every
        // lane walks the same generator so the group's shuffles line up
        uint32_t n_eff = 0;
        {
            const int n_cap = status == 0 ? min(a.n, a.n_off_cap) : 0;
            const int max_off = len - a.s;
            uint32_t used = 0;
            int level = 0, odd = -1, o = 0;
            bool active = false, done = n_cap == 0;
            auto next_off = [&]() -> int {
                for (;;) {
                    if (active) {
                        if (o <= max_off) {
                            const int v = o;
                            o += a.s;
                            return v;
                        }
                        active = false;
                    }
                    if (done) return -1;
                    int shift;
                    if (odd < 0) {
                        odd = 1;
                        level = 1;
                        shift = 0;
                    } else {
                        if ((1 << level) > 4 * a.s) {
                            done = true;
                            return -1;
                        }
                        shift = (odd * a.s) >> level;
                        odd += 2;
                        if (odd >= (1 << level)) {
                            ++level;
                            odd = 1;
                        }
                    }
                    if ((used >> shift) & 1u) continue;
                    used |= 1u << shift;
                    o = shift;
                    active = true;
                }
            };
            uint4* rec = live ? a.pre_recs + static_cast<uint64_t>(r) * a.pre_rstride : nullptr;
            int cnt = 0;
            // rounds of G seeds; the group agrees on when to stop
            for (;;) {
                int my_off = -1;
                int k = 0;
                if (status == 0 && len == tab_len) {  // the block's table (same list, same rounds)
                    const int rem = tab_n - cnt;
                    k = rem < 0 ? 0 : (rem < G ? rem : G);
                    if (g < k) my_off = s_off[cnt + g];
                } else {
                    for (; k < G; ++k) {
                        const int ov = cnt + k < n_cap ? next_off() : -1;
                        if (ov < 0) break;
                        if (k == g) my_off = ov;
                    }
                }
                const int round_n = __shfl_sync(gmask, k, gbase);  // same in every lane
                uint32_t l, h, n;
                fwd32(my_off >= 0 ? my_off : 0, l, h, n);
                if (my_off >= 0) {
                    uint4 rv;
                    if (n & seed_mask32(a.s)) {
                        rv = make_uint4(kSeedN, 0, 0, static_cast<uint32_t>(my_off));
                    } else {
                        const uint64_t key = planar_key(l, h, a.s);
                        const uint64_t rck = planar_rc_key(l, h, a.s);
                        const uint64_t canon = key < rck ? key : rck;
                        uint32_t fl = 0;
                        if (key != canon) fl |= kSeedQflip;
                        if (key == rck) fl |= kSeedPal;
                        if (a.eager > 0 && cnt + g >= a.eager) {
                            // beyond the eager seeds: probed on demand by the
                            // aligner (most reads stop after 2-4 lookups, C2 3.5)
                            rv = make_uint4(fl | kSeedLazy, static_cast<uint32_t>(canon),
                                            static_cast<uint32_t>(canon >> 32), static_cast<uint32_t>(my_off));
                        } else {
                            unsigned pl = 0, m = 0;
                            const bool found = probe_slot(a.table, a.n_slots, canon, pl, m);
                            uint32_t c = 0;
                            if (found) {
                                const uint32_t ntot = m & 0x7fffffffu;
                                c = (fl & kSeedPal) ? 2u * ntot : ntot;
                                if (m & 0x80000000u) fl |= kSeedSingleRc;
                            }
                            rv = make_uint4(fl, c, found ? pl : 0u, static_cast<uint32_t>(my_off));
                        }
                    }
                    rec[cnt + g] = rv;
                }
                cnt += round_n;
                // continue while any read of the warp still has seeds
                if (__ballot_sync(0xffffffffu, round_n == G && cnt < n_cap) == 0) break;
            }
            n_eff = static_cast<uint32_t>(cnt);
        }
        if (live && g == 0) a.pre_meta[r] = make_uint2(static_cast<uint32_t>(len), (status << 16) | n_eff);
    }
}

// L2 prefetch of the genome windows of a read's singleton seed hits (what
// seed_record does on the in-kernel path), one read ahead of its alignment.
SA_DEV void prefetch_windows(const AlignLaunch& a, const uint4* recs, int n, int len, int lane) {
    if (lane < n && lane < 32) {
        const uint4 rr = recs[lane];
        if (!(rr.x & (kSeedN | kSeedLazy)) && rr.y == 1u) {
            const uint32_t dir = ((rr.x & kSeedSingleRc) ? 1u : 0u) ^ ((rr.x & kSeedQflip) ? 1u : 0u);
            const int o = static_cast<int>(rr.w);
            const int64_t anc = static_cast<int64_t>(rr.z) - (dir ? (len - a.s - o) : o);
            const uint64_t b = anc < 0 ? 0 : (static_cast<uint64_t>(anc) >> 5);
            prefetch_l2(a.planes + b);
            prefetch_l2(a.planes + b + ((len + a.dl_max + 32) >> 5));
        }
    }
}


// kSlow: global candidate tables over a work list; kPipe: static striding with
// the cp.async read pipeline (short reads); kRegLV: register LV only;
// kStream: the pipelined kernel consumes a batch that is still being copied
// in (chunk flags; a separate variant so the default kernel carries none of it).
template <bool kSlow, bool kPipe, bool kRegLV, bool kStream = false, bool kPre = false>
__global__ void __launch_bounds__(32 * SA_FAST_WARPS, SA_MIN_BLOCKS) align_kernel(const AlignLaunch a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    unsigned char* ws = smem + static_cast<size_t>(wib) * a.smem_per_warp;

    // per-warp layout (capi.cu make_shape): planes[2] {R, C}, window, seed
    // records[2], probe landing zone, offsets[2], LV frontier, read staging[2],
    // stats, candidate table (global memory for the slow kernel)
    Ctx x;
    x.a = &a;
    x.lane = lane;
    // pruning-batch area at the end of the warp's share (capi.cu make_shape)
    unsigned char* pb = a.pb_on ? ws + a.smem_per_warp - kPbBytes : nullptr;
    // buffer q: R = planes + 2q*wbr, C = R + wbr (global slot per warp for the long-read layouts)
    // (only the dynamic-fetch kernel of reads > 1 kbp has global planes)
    const bool gpl = !kPipe && !kSlow && a.gplanes != nullptr;
    uint4* planes = gpl ? a.gplanes + static_cast<uint64_t>((blockIdx.x * blockDim.x + threadIdx.x) >> 5) *
                                          a.gplanes_per_warp
                        : reinterpret_cast<uint4*>(ws);
    // one {R, C} buffer without the read pipeline
    x.W = gpl ? reinterpret_cast<uint4*>(ws) : planes + (a.prefetch ? 4 : 2) * a.wbr;
    uint4* recs = x.W + (a.gw ? 0 : a.wbw);  // 2 x 32; no window area when the LV reads the genome in place
    uint4* pslot = recs + 64;                       // 32
    unsigned long long* pcanon = reinterpret_cast<unsigned long long*>(pslot + 32);  // 32
    int* offs = reinterpret_cast<int*>(pcanon + 32);  // 2 x n_off_cap
    x.F = offs + 2 * a.n_off_cap;
    x.qbm = !kRegLV && a.f_ints * 32 >= (1 << (2 * kQfQ)) ? reinterpret_cast<uint32_t*>(x.F) : nullptr;
    uint32_t* stage = reinterpret_cast<uint32_t*>(x.F + a.f_ints);  // 2 x sbw words
    // warp totals, lane-distributed (lane k: sa_stats slot k); LV cells per lane
    unsigned long long acc = 0;
    x.cells = 0;
    x.qf_tries = 0;
    x.qf_hits = 0;
    unsigned char* tb;
    if (kSlow) {
        const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
        tb = a.gscratch + gw * a.gscratch_per_warp;
    } else {
        tb = reinterpret_cast<unsigned char*>(reinterpret_cast<unsigned long long*>(stage + 2 * a.sbw) + kNumStats);
    }
    x.t.cap = a.cap;
    x.t.hcap = a.hcap;
    x.t.ckey = reinterpret_cast<unsigned long long*>(tb);
    x.t.cmask = x.t.ckey + a.cap;
    x.t.hkey = x.t.cmask + a.cap;
    x.t.ccnt = reinterpret_cast<uint32_t*>(x.t.hkey + a.hcap);
    x.t.chslot = x.t.ccnt + a.cap;
    x.t.hval = x.t.chslot + a.cap;
    // the global tables of the overflow kernel are cleared by a warp only when
    // it gets work (usually none: the launch follows every device batch)
    bool table_ready = !kSlow;
    if (!kSlow) {
        for (int j = lane; j < a.hcap; j += 32) x.t.hkey[j] = kEmptyKey;
        __syncwarp();
    }

    int cached_len0 = -1, cached_len1 = -1, n_eff0 = 0, n_eff1 = 0;
    // offsets for read length len into buffer q (cached per buffer)
    auto offsets_for = [&](int q, int len) -> int {
        int& cl = q ? cached_len1 : cached_len0;
        int& ne = q ? n_eff1 : n_eff0;
        if (len != cl) {
            ne = compute_offsets(len, a.s, min(a.n, a.n_off_cap), offs + q * a.n_off_cap, lane);
            cl = len;
        }
        return ne;
    };
    auto bad_read = [&](uint32_t r) {
        if (lane == 0) {
            atomicOr(a.error_flag, 1u);
            atomicMin(a.error_read, a.read_base + r);
        }
    };
    auto short_read = [&](uint32_t r, int len) {  // REF aligner.cpp:231-235
        if (lane == 0) {
            sa_result res;
            res.position = 0;
            res.distance = -1;
            res.gap = 0;
            res.kind = SA_NOT_FOUND;
            res.has_position = 0;
            res.direction = 0;
#pragma unroll
            for (int i = 0; i < 5; ++i) res.reserved[i] = 0;
            a.results[r] = res;
        }
        acc += (lane == S_READS || lane == S_TOO_SHORT || lane == S_NOT_FOUND) ? 1u
               : (lane == S_READ_BASES ? static_cast<uint32_t>(len) : 0u);
    };
    auto overflowed = [&](uint32_t r) {
        if (kSlow) {  // table sized n_eff * h_max cannot overflow unless clamped
            if (lane == 0) atomicOr(a.error_flag, 2u);
        } else if (lane == 0) {  // defer to the global-table kernel
            const unsigned slot = atomicAdd(a.overflow_count, 1u);
            a.overflow_list[slot] = static_cast<unsigned>(a.read_base) + r;  // batch-absolute id
        }
        if (!kSlow && lane == S_OVERFLOW) acc += 1u;
    };
    // status of a staged read: 0 = decoded, 1 = shorter than s, 2 = bad character
    auto prep = [&](int q, int len, const uint32_t* words, int sh, int nwd) -> int {
        if (len < a.s) return 1;
        if (len > a.lcap) return 3;  // beyond this launch's layout: deferred
        offsets_for(q, len);
        uint4* R = planes + 2 * q * a.wbr;
        return decode_read(words, sh, nwd, len, R, R + a.wbr, lane) ? 2 : 0;
    };
    auto process = [&](uint32_t r, int q, int len, int st, bool wave0_ready, int ne_pre = -1,
                       const uint4* grecs = nullptr) {
        if (st == 1) {
            short_read(r, len);
        } else if (st == 2) {
            bad_read(r);
        } else if (st == 3) {
            overflowed(r);
        } else {
            x.R = planes + 2 * q * a.wbr;
            x.C = x.R + a.wbr;
            x.len = len;
            x.d_max = a.dmax_param >= 0 ? a.dmax_param : (12 * len + 99) / 100;
            const int ne = ne_pre >= 0 ? ne_pre : (q ? n_eff1 : n_eff0);
            if (align_one<kRegLV, kSlow, !kPipe && !kSlow && !kRegLV>(x, r, ne, offs + q * a.n_off_cap, len / a.s, acc, recs + 32 * q, wave0_ready,
                                  grecs, pb) == 0)
                overflowed(r);
        }
    };

    if (kPre) {
        // Two-kernel path: planes and seed records come from seed_kernel.
        // Static striding, one read ahead: while read r is aligned, the
        // planes and wave-0 records of read r+nw are copied into the other
        // buffer (cp.async) and its singleton windows are prefetched to L2.
        const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
        // after solo_kernel: only the reads it left in pre_list
        const bool listed = a.pre_list != nullptr;
        const uint32_t N = listed ? *a.pre_list_count : a.n_reads;
        const int half = a.pre_pstride >> 1;
        const int nrec = min(32, a.pre_rstride);
        auto rid = [&](uint32_t k) -> uint32_t { return listed ? __ldg(a.pre_list + k) : k; };
        auto issue_copy = [&](uint32_t rr, int q) {
            rr = rid(rr);
            const uint4* gp = a.pre_planes + static_cast<uint64_t>(rr) * a.pre_pstride;
            uint4* R = planes + 2 * q * a.wbr;
            for (int t = lane; t < half; t += 32) {
                cp_async16(R + t, gp + t);
                cp_async16(R + a.wbr + t, gp + half + t);
            }
            const uint4* gr = a.pre_recs + static_cast<uint64_t>(rr) * a.pre_rstride;
            for (int t = lane; t < nrec; t += 32) cp_async16(recs + 32 * q + t, gr + t);
        };
        // Reads are fetched dynamically (a.work_cursor, zeroed by the seed
        // kernel), one read ahead: listed reads vary widely in cost, and with
        // static striding a launch lasted as long as its unluckiest warp
        // (chunks of the batch pipeline hold ~20 listed reads per warp).
        // Without a cursor (never in practice) reads are strided statically.
        const bool dyn = a.work_cursor != nullptr;
        uint32_t stat_next = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        auto grab = [&]() -> uint32_t {
            uint32_t v;
            if (dyn) {
                v = 0;
                if (lane == 0) v = atomicAdd(a.work_cursor, 1u);
                v = __shfl_sync(FULL, v, 0);
            } else {
                v = stat_next;
                stat_next += nw;
            }
            return v;
        };
        uint32_t r = grab();
        if (r < N) {
            uint2 m_c = __ldg(a.pre_meta + rid(r)), m_n = make_uint2(0, 1u << 16);
            issue_copy(r, 0);
            cp_async_commit();
            uint32_t r_n = grab();
            if (r_n < N) {
                m_n = __ldg(a.pre_meta + rid(r_n));
                issue_copy(r_n, 1);
            }
            cp_async_commit();
            int p = 0;
            while (r < N) {
                cp_async_wait0();  // read r (and r_n, issued an iteration ago) have landed
                __syncwarp();
                if (r_n < N && (m_n.y >> 16) == 0)
                    prefetch_windows(a, recs + 32 * (p ^ 1), static_cast<int>(m_n.y & 0xffffu),
                                     static_cast<int>(m_n.x), lane);
                const uint32_t r_nn = r_n < N ? grab() : N;
                uint2 m_nn = make_uint2(0, 1u << 16);
                if (r_nn < N) m_nn = __ldg(a.pre_meta + rid(r_nn));
                const uint32_t rr = rid(r);
                process(rr, p, static_cast<int>(m_c.x), static_cast<int>(m_c.y >> 16), true,
                        static_cast<int>(m_c.y & 0xffffu), a.pre_recs + static_cast<uint64_t>(rr) * a.pre_rstride);
                if (r_nn < N) issue_copy(r_nn, p);
                cp_async_commit();
                m_c = m_n;
                m_n = m_nn;
                r = r_n;
                r_n = r_nn;
                p ^= 1;
            }
            cp_async_wait0();
        }
    } else if (kPipe) {
        // Static striding, software-pipelined one read ahead: while read r is
        // aligned, read r+nw is already decoded and its wave-0 index probes are
        // in flight (cp.async), and read r+2nw's bytes are being copied.
        const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
        const uint32_t N = a.n_reads;
        constexpr bool stream = kStream;
        uint32_t ready_c = 0;  // streaming: chunks below this are known resident
        // Chunks land in order; wait (lane 0 polls) until read rr's chunk has.
        // A flag that never arrives times out into an error instead of a hang.
        auto wait_chunk = [&](uint32_t rr) {
            if (!stream) return;
            const uint32_t c = stream_chunk_of(rr, a.chunk_shift0, a.chunk_shift);
            if (c < ready_c) return;
            if (lane == 0) {
                const volatile unsigned int* f = a.chunk_flag + c;
                const long long t0 = clock64();
                while (*f != a.epoch) {
                    __nanosleep(256);
                    if (clock64() - t0 > (1ll << 35)) {
                        atomicOr(a.error_flag, 4u);
                        break;
                    }
                }
            }
            __syncwarp();
            ready_c = c + 1;
        };
        // offsets are read from L2 (.cg): a line may hold a neighbour chunk's
        // entries that landed after this SM cached it
        auto off = [&](uint32_t i) -> uint64_t {
            return stream ? __ldcg(reinterpret_cast<const unsigned long long*>(a.offsets) + i) : a.offsets[i];
        };
        auto raddr = [&](uint32_t rr, uint64_t o) -> const char* {
            return stream ? a.bases + (static_cast<long long>(o) + __ldcg(a.chunk_adj + stream_chunk_of(rr, a.chunk_shift0, a.chunk_shift)))
                          : a.bases + (o - a.base_off);
        };
        // finished reads are counted per warp and published once per chunk
        // (one fence + atomic per warp and chunk, not per read)
        uint32_t done_c = 0, done_n = 0;
        auto flush_done = [&]() {
            if (done_n && lane == 0) {
                __threadfence();
                atomicAdd(a.chunk_done + done_c, done_n);
            }
            done_n = 0;
        };
        auto read_done = [&](uint32_t rr) {
            if (!stream) return;
            const uint32_t c = stream_chunk_of(rr, a.chunk_shift0, a.chunk_shift);
            if (c != done_c) {
                flush_done();
                done_c = c;
            }
            ++done_n;
        };
        auto copy_read = [&](uint32_t rr, uint64_t o0, uint64_t o1, uint32_t* dst, int& sh, int& nwd) {
            const int len = static_cast<int>(o1 - o0);
            if (len > a.lcap) {  // not staged; prep() defers it
                sh = 0;
                nwd = 0;
                return;
            }
            issue_read_copy(raddr(rr, o0), len, dst, lane, sh, nwd);
        };
        uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        if (r < N) {
            wait_chunk(r);
            const uint64_t c0 = off(r), c1 = off(r + 1);
            uint64_t n0 = 0, n1 = 0;
            if (r + nw < N) {
                wait_chunk(r + nw);
                n0 = off(r + nw);
                n1 = off(r + nw + 1);
            }
            int sh = 0, nwd = 0;
            copy_read(r, c0, c1, stage, sh, nwd);
            cp_async_commit();
            cp_async_wait0();
            __syncwarp();
            int len_cur = static_cast<int>(c1 - c0);
            int st_cur = prep(0, len_cur, stage, sh, nwd);
            if (st_cur == 0) {
                issue_wave0(a, planes, offs, n_eff0, recs, pslot, pcanon, lane);
                resolve_wave0(a, n_eff0, len_cur, recs, pslot, pcanon, lane);
            }
            int sh_n = 0, nw_n = 0;
            if (r + nw < N) copy_read(r + nw, n0, n1, stage + a.sbw, sh_n, nw_n);
            cp_async_commit();
            int p = 0;
            for (; r < N; r += nw) {
                const bool has_next = r + nw < N;
                const bool has_next2 = r + 2 * nw < N;
                cp_async_wait0();
                __syncwarp();
                const int len_n = static_cast<int>(n1 - n0);
                int st_n = 1;
                if (has_next) {
                    st_n = prep(p ^ 1, len_n, stage + (p ^ 1) * a.sbw, sh_n, nw_n);
                    if (st_n == 0)
                        issue_wave0(a, planes + 2 * (p ^ 1) * a.wbr, offs + (p ^ 1) * a.n_off_cap,
                                    p ? n_eff0 : n_eff1, recs + 32 * (p ^ 1), pslot, pcanon, lane);
                }
                uint64_t f0 = 0, f1 = 0;
                if (has_next2) {
                    wait_chunk(r + 2 * nw);
                    f0 = off(r + 2 * nw);
                    f1 = off(r + 2 * nw + 1);
                }
                process(r, p, len_cur, st_cur, true);
                read_done(r);
                if (has_next && st_n == 0)
                    resolve_wave0(a, p ? n_eff0 : n_eff1, len_n, recs + 32 * (p ^ 1), pslot, pcanon, lane);
                sh_n = 0;
                nw_n = 0;
                if (has_next2) copy_read(r + 2 * nw, f0, f1, stage + p * a.sbw, sh_n, nw_n);
                cp_async_commit();
                n0 = f0;
                n1 = f1;
                len_cur = len_n;
                st_cur = st_n;
                p ^= 1;
            }
            cp_async_wait0();
            flush_done();
        }
    } else {
        // dynamic fetch (work list for the slow kernel), reads decoded from global
        const uint32_t n_work = kSlow ? *a.work_count : a.n_reads;
        for (;;) {
            uint32_t r = 0;
            if (lane == 0) r = atomicAdd(a.cursor, 1u);
            r = __shfl_sync(FULL, r, 0);
            if (r >= n_work) break;
            if (!table_ready) {
                for (int j = lane; j < a.hcap; j += 32) x.t.hkey[j] = kEmptyKey;
                __syncwarp();
                table_ready = true;
            }
            // the list holds launch-absolute ids (read_base + r, as overflowed() stores
            // them); no list: every read of the launch
            if (kSlow && a.work_list) r = a.work_list[r] - static_cast<uint32_t>(a.read_base);
            uint64_t o0, o1;
            if (a.fixed_len) {  // equal-length chunk: no offsets were copied in
                o0 = a.base_off + static_cast<uint64_t>(r) * a.fixed_len;
                o1 = o0 + a.fixed_len;
            } else {
                o0 = a.offsets[r];
                o1 = a.offsets[r + 1];
            }
            const int len = static_cast<int>(o1 - o0);
            const uintptr_t addr = reinterpret_cast<uintptr_t>(a.bases + (o0 - a.base_off));
            const uintptr_t abase = addr & ~static_cast<uintptr_t>(3);
            const int nwords = static_cast<int>((addr + len - abase + 3) >> 2);
            const int st = prep(0, len, reinterpret_cast<const uint32_t*>(abase), static_cast<int>(addr & 3), nwords);
            process(r, 0, len, st, false);
        }
    }

    __syncwarp();
    unsigned long long cells = x.cells;
    for (int o = 16; o > 0; o >>= 1) cells += __shfl_xor_sync(FULL, cells, o);
    if (lane == S_CELLS) acc += cells;
    if (lane < kNumStats && acc) atomicAdd(a.stats + lane, acc);
}

// The prune queue's reads (pq_defer): warp per read, a persistent grid.
__global__ void __launch_bounds__(256) prune_kernel(const AlignLaunch a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    constexpr uint32_t kTab = 64 * (8 + 8 + 4);
    const uint32_t planes_bytes = static_cast<uint32_t>(a.pre_pstride) * 16u;
    unsigned char* ws = smem + static_cast<size_t>(wib) * (kTab + kPbBytes + planes_bytes);
    uint4* planes = reinterpret_cast<uint4*>(ws + kTab + kPbBytes);
    Ctx x;
    x.a = &a;
    x.lane = lane;
    x.cells = 0;
    x.qf_tries = 0;
    x.qf_hits = 0;
    x.qbm = nullptr;  // (the pruning batch holds its own LV)
    x.t.cap = 64;
    x.t.hcap = 0;
    x.t.ckey = reinterpret_cast<unsigned long long*>(ws);
    x.t.cmask = x.t.ckey + 64;
    x.t.ccnt = reinterpret_cast<uint32_t*>(x.t.cmask + 64);
    x.t.chslot = nullptr;
    x.t.hkey = nullptr;
    x.t.hval = nullptr;
    unsigned char* pb = ws + kTab;
    const int half = a.pre_pstride >> 1;
    unsigned long long acc = 0;
    const uint32_t n = *a.pq_count;
    for (;;) {
        uint32_t k = 0;
        if (lane == 0) k = atomicAdd(a.pq_cursor2, 1u);
        k = __shfl_sync(FULL, k, 0);
        if (k >= n) break;
        const unsigned char* rec = a.pq_pool + (static_cast<uint64_t>(__ldg(a.pq_list + k)) << 4);
        const uint32_t* h = reinterpret_cast<const uint32_t*>(rec);
        const uint32_t r = h[0];
        x.len = static_cast<int>(h[1]);
        x.tr.d_best = static_cast<int>(h[2]);
        x.tr.d_second = static_cast<int>(h[3]);
        x.tr.best_pos = reinterpret_cast<const uint64_t*>(rec)[2];
        x.first_pos = reinterpret_cast<const uint64_t*>(rec)[3];
        x.calls = h[8];
        x.n_cands = h[9];
        x.n_unscored = h[10];
        const uint32_t fl = h[11];
        x.d_max = static_cast<int>(h[12]);
        const int B = static_cast<int>(h[13]);
        x.first_done = (fl & PQ_FIRST_DONE) != 0;
        x.first_valid = (fl & PQ_FIRST_VALID) != 0;
        x.first_dir = (fl & PQ_FIRST_DIR) ? 1 : 0;
        x.tr.best_dir = (fl & PQ_BEST_DIR) ? 1 : 0;
        x.rs = lane < kNumStats ? reinterpret_cast<const uint32_t*>(rec + 64)[lane] : 0u;
        const unsigned long long* keys = reinterpret_cast<const unsigned long long*>(rec + kPqHeader);
        for (uint32_t j = lane; j < x.n_cands; j += 32) {
            x.t.ckey[j] = keys[j];
            x.t.cmask[j] = keys[x.n_cands + j];
            x.t.ccnt[j] = reinterpret_cast<const uint32_t*>(keys + 2 * x.n_cands)[j];
        }
        {  // the read's forward and reverse-complement planes, into shared memory
            const uint4* gp = a.pre_planes + static_cast<uint64_t>(r) * a.pre_pstride;
            for (int t = lane; t < a.pre_pstride; t += 32) planes[t] = gp[t];
        }
        x.R = planes;
        x.C = planes + half;
        __syncwarp();
        bool early_multi = false;
        if (prune_all(x, pb, B)) {
            stat_add(x, S_MULTI, 1u);
            early_multi = true;
        }
        finish_read(x, r, early_multi, (fl & PQ_ANY_POP) != 0, (fl & PQ_ANY_LOOKUP) != 0, acc);
    }
    __syncwarp();
    unsigned long long cells = x.cells;
    for (int o = 16; o > 0; o >>= 1) cells += __shfl_xor_sync(FULL, cells, o);
    if (lane == S_CELLS) acc += cells;
    if (lane < kNumStats && acc) atomicAdd(a.stats + lane, acc);
}

// ------------------------------------------------------------------ standalone LV

__global__ void __launch_bounds__(256) lv_batch_kernel(const LvLaunch a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    unsigned char* ws = smem + static_cast<size_t>(wib) * a.smem_per_warp;
    uint4* R = reinterpret_cast<uint4*>(ws);
    uint4* W = R + a.wbr;
    int* F = reinterpret_cast<int*>(W + a.wbw);
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t p = gw; p < a.n_pairs; p += nw) {
        const int m = static_cast<int>(a.read_off[p + 1] - a.read_off[p]);
        const int w = static_cast<int>(a.win_off[p + 1] - a.win_off[p]);
        const char* rs = a.reads + a.read_off[p];
        const char* wsrc = a.wins + a.win_off[p];
        int dl = a.d_limits[p];
        // distance <= m always (m insertions), so a limit above m changes nothing
        if (dl > m) dl = m;
        bool bad = false;
        const int rb = (m + 31) / 32 + 1, wb = (w + 31) / 32 + 1;
        for (int b = 0; b < rb; ++b) {
            const int pos = b * 32 + lane;
            const int code = pos < m ? read_code(static_cast<unsigned char>(rs[pos])) : 4;
            bad |= code == 5;
            const uint32_t lo = __ballot_sync(FULL, code < 4 && (code & 1));
            const uint32_t hi = __ballot_sync(FULL, code < 4 && (code & 2));
            const uint32_t nn = __ballot_sync(FULL, code >= 4);
            if (lane == 0) R[b] = make_uint4(lo, hi, nn, 0);
        }
        for (int b = 0; b < wb; ++b) {
            const int pos = b * 32 + lane;
            const int code = pos < w ? read_code(static_cast<unsigned char>(wsrc[pos])) : 4;
            bad |= code == 5;
            const uint32_t lo = __ballot_sync(FULL, code < 4 && (code & 1));
            const uint32_t hi = __ballot_sync(FULL, code < 4 && (code & 2));
            const uint32_t nn = __ballot_sync(FULL, code >= 4);
            if (lane == 0) W[b] = make_uint4(lo, hi, nn, 0);
        }
        __syncwarp();
        if (__any_sync(FULL, bad)) {
            if (lane == 0) {
                atomicOr(a.error_flag, 1u);
                a.out[p] = -2;
            }
            continue;
        }
        uint32_t cells = 0;
        if (a.bitpar == 1 && dl <= 15) {  // test hook: the solo kernel's bit-parallel LV, lane 0 alone
            if (lane == 0) a.out[p] = lv_bitpar(R, rb, m, W, 0u, w, dl, cells);
            __syncwarp();
            continue;
        }
        const int d = lv_warp_any(R, m, W, 0u, w, dl, F, lane, cells, a.bitpar_min, a.bitpar == 2);
        if (lane == 0) a.out[p] = d;
        __syncwarp();
    }
}

// ------------------------------------------------------------------ lookup

// SeedIndex::lookup over a batch (REF src/seed_index.cpp:128-143), one thread
// per seed.  Seeds are ASCII; anything but A/C/G/T (any case) yields 0 hits
// like pack_seed's failure path (REF :51-60, :141).
__global__ void lookup_kernel(const LookupLaunch a) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < a.n_seeds;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const char* sd = a.seeds + i * a.s;
        uint32_t lo = 0, hi = 0;
        bool ok = true;
        for (int j = 0; j < a.s; ++j) {
            int b;
            switch (sd[j]) {
                case 'A': case 'a': b = 0; break;
                case 'C': case 'c': b = 1; break;
                case 'G': case 'g': b = 2; break;
                case 'T': case 't': b = 3; break;
                default: b = -1;
            }
            if (b < 0) ok = false;
            lo |= static_cast<uint32_t>(b & 1) << j;
            hi |= static_cast<uint32_t>((b >> 1) & 1) << j;
        }
        uint32_t nf = 0, nr = 0;
        if (ok) {
            const uint64_t key = planar_key(lo, hi, a.s);
            const uint64_t rc = planar_rc_key(lo, hi, a.s);
            const uint64_t canon = key < rc ? key : rc;
            const bool qflip = key != canon, pal = key == rc;
            unsigned int payload, meta;
            if (probe_slot(a.table, a.n_slots, canon, payload, meta)) {
                const uint32_t ntot = meta & 0x7fffffffu;
                uint32_t n_canon;  // windows equal to canon
                if (ntot == 1) n_canon = (meta & 0x80000000u) ? 0u : 1u;
                else n_canon = a.pool[payload];
                auto pos_at = [&](uint32_t j) -> uint64_t {
                    return ntot == 1 ? payload : a.pool[payload + 1 + j];
                };
                if (pal) {
                    nf = nr = ntot;
                    if (a.fwd_out)
                        for (uint32_t j = 0; j < ntot && j < a.cap; ++j) {
                            a.fwd_out[i * a.cap + j] = pos_at(j);
                            a.rc_out[i * a.cap + j] = pos_at(j);
                        }
                } else {
                    // forward list = windows equal to the query
                    const uint32_t fb = qflip ? n_canon : 0, fe = qflip ? ntot : n_canon;
                    const uint32_t rb = qflip ? 0 : n_canon, re = qflip ? n_canon : ntot;
                    nf = fe - fb;
                    nr = re - rb;
                    if (a.fwd_out) {
                        for (uint32_t j = 0; j < nf && j < a.cap; ++j)
                            a.fwd_out[i * a.cap + j] = pos_at(fb + j);
                        for (uint32_t j = 0; j < nr && j < a.cap; ++j)
                            a.rc_out[i * a.cap + j] = pos_at(rb + j);
                    }
                }
            }
        }
        a.counts[i] = nf + nr;
        if (a.n_fwd) a.n_fwd[i] = nf;
        if (a.n_rc) a.n_rc[i] = nr;
    }
}

}  // namespace

template <bool kSlow, bool kPipe, bool kRegLV, bool kStream = false, bool kPre = false>
void launch_variant(const AlignLaunch& a, int grid, int block, cudaStream_t st) {
    align_kernel<kSlow, kPipe, kRegLV, kStream, kPre><<<grid, block, a.smem_per_warp * (block / 32), st>>>(a);
}

// kernel variants: fast {pipelined, streamed, dynamic} x {register LV, shared LV}; slow {register, shared}
template <bool kSlow, bool kPipe, bool kRegLV, bool kStream = false, bool kPre = false>
cudaError_t set_smem_variant(int bytes) {
    return cudaFuncSetAttribute(align_kernel<kSlow, kPipe, kRegLV, kStream, kPre>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

void launch_align_fast(const AlignLaunch& a, int grid, int block, cudaStream_t st) {
    const bool reg = a.dl_max <= 15;
    if (a.prefetch && a.chunk_flag) {
        if (reg) launch_variant<false, true, true, true>(a, grid, block, st);
        else launch_variant<false, true, false, true>(a, grid, block, st);
    } else if (a.prefetch) {
        if (reg) launch_variant<false, true, true>(a, grid, block, st);
        else launch_variant<false, true, false>(a, grid, block, st);
    } else {
        if (reg) launch_variant<false, false, true>(a, grid, block, st);
        else launch_variant<false, false, false>(a, grid, block, st);
    }
}

bool solo_eligible(const AlignLaunch& a);

void launch_seed(const AlignLaunch& a0, cudaStream_t st) {
    // lazy seeds only where the solo kernel runs (it probes them on demand and
    // resolves the rest of the reads it lists, resolve_kernel); a launch on the
    // warp kernel alone gets every seed probed here
    AlignLaunch a = a0;
    if (!solo_eligible(a)) a.eager = 0;
    // G lanes per read: the smallest power of two covering the blocks
    const int nbmax = (a.pre_pstride >> 1) - 1;
    auto go = [&](auto kernel, int G) {
        const uint64_t groups_per_block = 256 / G;
        uint64_t g = (static_cast<uint64_t>(a.n_reads) + groups_per_block - 1) / groups_per_block;
        static const uint64_t cap = [] {  // SA_SEED_GRID overrides (tuning)
            const char* e = getenv("SA_SEED_GRID");
            // 64 blocks per SM, grid-stride beyond: a block lists the seed offsets once for its reads
            // (a group per read -- 2^23 blocks -- measured 491 M reads/s at C2 against 497 M)
            return e ? static_cast<uint64_t>(atoll(e)) : uint64_t{148 * 64};
        }();
        // gridDim.x * blockDim.x is a 32-bit product in the kernel: at most 2^31 threads
        g = std::max<uint64_t>(1, std::min<uint64_t>({g, std::max<uint64_t>(cap, 1), uint64_t{1} << 23}));
        kernel<<<static_cast<int>(g), 256, 0, st>>>(a);
    };
    if (nbmax <= 4) go(seed_kernel<4>, 4);
    else if (nbmax <= 8) go(seed_kernel<8>, 8);
    else if (nbmax <= 16) go(seed_kernel<16>, 16);
    else go(seed_kernel<32>, 32);
}

// Small launches stay on the warp kernel: with one read per thread a launch
// of a few thousand reads is as long as its slowest read (C0, 10 k reads:
// 135 M reads/s with the solo kernel, 171 M without).  SA_SOLO_MIN_READS
// overrides the threshold; SA_NO_SOLO switches the solo kernel off.
bool solo_eligible(const AlignLaunch& a) {
    static const bool off = getenv("SA_NO_SOLO") != nullptr;
    static const uint32_t min_reads = [] {
        const char* e = getenv("SA_SOLO_MIN_READS");
        return e ? static_cast<uint32_t>(atoll(e)) : 12288u;
    }();
    // the solo kernel keys candidates as 32-bit (bucket << 1 | dir): buckets
    // must stay below 2^31 (bucket_size 1 on a genome past 2^31 bases would
    // fold anchors a and a + 2^31 together)
    return !off && a.pre_list != nullptr && a.n_reads >= min_reads && a.dl_max <= 15 && a.bs_shift >= 0 &&
           a.bs_shift <= 5 && (a.glen >> a.bs_shift) < (1ull << 31);
}

// Diagnostics (SA_DEBUG_KTIME): per-kernel device time of the kPre launches,
// accumulated; sab_debug_ktimes prints and resets them (serialises the stream).
namespace {
struct KTimer {
    bool on = getenv("SA_DEBUG_KTIME") != nullptr;
    double ms[4] = {0, 0, 0, 0};  // solo, resolve, warp, prune
    cudaEvent_t ev[5] = {};
    void mark(int i, cudaStream_t st) {
        if (!on) return;
        if (!ev[i]) cudaEventCreate(&ev[i]);
        cudaEventRecord(ev[i], st);
    }
    void span(int k, int i0, int i1) {
        if (!on) return;
        cudaEventSynchronize(ev[i1]);
        float t = 0;
        cudaEventElapsedTime(&t, ev[i0], ev[i1]);
        ms[k] += t;
    }
};
KTimer& ktimer() {
    static KTimer t;
    return t;
}
}  // namespace

// Diagnostics (SA_DEBUG_TIMELINE, capi.cu): called after each kernel of a
// seeded launch with a tag (o solo, r resolve, w warp, p prune) and its stream.
thread_local void (*g_timeline_hook)(char tag, cudaStream_t st) = nullptr;

extern "C" void sab_debug_ktimes(const char* tag) {
    KTimer& t = ktimer();
    if (!t.on) return;
    fprintf(stderr, "[ktime] %s solo %.3f resolve %.3f warp %.3f prune %.3f ms\n", tag, t.ms[0], t.ms[1], t.ms[2],
            t.ms[3]);
    for (double& m : t.ms) m = 0;
}

int launch_align_seeded(const AlignLaunch& a, int grid, int block, cudaStream_t st) {
    KTimer& kt = ktimer();
    kt.mark(0, st);
    AlignLaunch b = a;
    int n = 1;
    if (solo_eligible(a)) {
        static const uint64_t cap = [] {  // blocks (grid-stride beyond); SA_SOLO_GRID overrides
            const char* e = getenv("SA_SOLO_GRID");
            return e ? static_cast<uint64_t>(atoll(e)) : 148ull * SA_SOLO_MIN_BLOCKS;  // one resident wave (C1 992 -> 1018 M)
        }();
        const uint64_t g = std::min<uint64_t>((static_cast<uint64_t>(a.n_reads) + kSoloThreads - 1) / kSoloThreads,
                                              std::max<uint64_t>(cap, 1));
        static const bool dbg = getenv("SA_DEBUG_SOLO") != nullptr;  // diagnostics: reads left to the warp kernel
        static unsigned int* d_dbg = nullptr;
        AlignLaunch sa = a;
        if (dbg) {
            if (!d_dbg) cudaMalloc(&d_dbg, 4 * sizeof(unsigned int));
            cudaMemsetAsync(d_dbg, 0, 4 * sizeof(unsigned int), st);
            sa.dbg = d_dbg;
        }
        solo_kernel<<<static_cast<int>(std::max<uint64_t>(g, 1)), kSoloThreads, 0, st>>>(sa);
        ++n;
        kt.mark(1, st);
        if (g_timeline_hook) g_timeline_hook('o', st);
        kt.span(0, 0, 1);
        if (a.eager > 0 && a.eager < a.n) {  // lazy records of the listed reads
            resolve_kernel<<<148 * 8, 256, 0, st>>>(a);
            ++n;
            kt.mark(2, st);
            if (g_timeline_hook) g_timeline_hook('r', st);
            kt.span(1, 1, 2);
            kt.mark(1, st);
        }
        if (dbg) {
            unsigned int n = 0, why[4] = {0, 0, 0, 0};
            cudaStreamSynchronize(st);
            cudaMemcpy(&n, a.pre_list_count, sizeof(n), cudaMemcpyDeviceToHost);
            cudaMemcpy(why, d_dbg, sizeof(why), cudaMemcpyDeviceToHost);
            fprintf(stderr, "[solo] %u of %u reads to the warp kernel (hits %u, candidates %u, long LV %u)\n", n,
                    a.n_reads, why[0], why[1], why[2]);
        }
    } else {
        b.pre_list = nullptr;
        b.pre_list_count = nullptr;
    }
#if SA_DEBUG_COUNTERS
    static unsigned int* d_wdbg = nullptr;
    if (!d_wdbg) {
        cudaMalloc(&d_wdbg, 16 * sizeof(unsigned int));
    }
    cudaMemsetAsync(d_wdbg, 0, 16 * sizeof(unsigned int), st);
    b.dbg = d_wdbg;
#endif
    // nothing is deferred without the pruning batch, nor in launches too small
    // for the solo kernel (C0, 10 k reads: the extra launch costs more than it saves)
    if (!b.pb_on || !solo_eligible(a)) b.pq_pool = nullptr;
    kt.mark(2, st);
    if (b.dl_max <= 15) launch_variant<false, true, true, false, true>(b, grid, block, st);
    else launch_variant<false, true, false, false, true>(b, grid, block, st);
    kt.mark(3, st);
    if (g_timeline_hook) g_timeline_hook('w', st);
    kt.span(2, 2, 3);
    if (b.pq_pool) {  // the reads it handed to the prune queue
        const uint32_t spw = prune_kernel_smem_per_warp() + static_cast<uint32_t>(b.pre_pstride) * 16u;
        static uint32_t attr = 0;
        if (attr < 8 * spw) {
            cudaFuncSetAttribute(prune_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * spw);
            attr = 8 * spw;
        }
        prune_kernel<<<148 * 4, 256, 8 * spw, st>>>(b);
        ++n;
        kt.mark(4, st);
        if (g_timeline_hook) g_timeline_hook('p', st);
        kt.span(3, 3, 4);
    }
#if SA_DEBUG_COUNTERS
    {
        unsigned int h[16];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, d_wdbg, sizeof(h), cudaMemcpyDeviceToHost);
        fprintf(stderr, "[warp] reads %u: seed-loop LV calls %u iterations %u d_limit sum %u; pruning entries %u "
                        "candidates %u B sum %u\n", a.pre_list_count ? 0u : a.n_reads, h[4], h[5], h[6], h[7], h[8], h[9]);
    }
#endif
    return n;
}

int launch_align_pre(const AlignLaunch& a, int grid, int block, cudaStream_t st) {
    launch_seed(a, st);
    return 1 + launch_align_seeded(a, grid, block, st);
}

void launch_align_slow(const AlignLaunch& a0, int grid, int block, cudaStream_t st) {
    AlignLaunch a = a0;
    a.gplanes = nullptr;  // its own grid: planes in shared memory (slow_smem_per_warp holds them)
    if (a.dl_max <= 15) launch_variant<true, false, true>(a, grid, block, st);
    else launch_variant<true, false, false>(a, grid, block, st);
}

void launch_lv_batch(const LvLaunch& a, int grid, int block, cudaStream_t st) {
    // test hooks: SA_LV_BITPAR (lv_bitpar for d_limit <= 15), SA_LV_LONG=bitpar (lv_bitpar_warp
    // instead of the systolic lv_sys for the long-read limits)
    static const int bitpar = getenv("SA_LV_BITPAR") != nullptr
                                  ? 1
                                  : (getenv("SA_LV_LONG") && !strcmp(getenv("SA_LV_LONG"), "bitpar") ? 2 : 0);
    static const int bitpar_min = [] {  // test hook: the warp bit-parallel LV from this limit
        const char* e = getenv("SA_LV_WARP_BITPAR_MIN");
        return e ? std::max(16, atoi(e)) : SA_BITPAR_MIN_DL;
    }();
    LvLaunch b = a;
    b.bitpar = bitpar;
    b.bitpar_min = bitpar_min;
    lv_batch_kernel<<<grid, block, b.smem_per_warp * (block / 32), st>>>(b);
}

void launch_lookup(const LookupLaunch& a, cudaStream_t st) {
    uint64_t g = (a.n_seeds + 127) / 128;
    if (g > 148 * 32) g = 148 * 32;
    if (g < 1) g = 1;
    lookup_kernel<<<static_cast<int>(g), 128, 0, st>>>(a);
}

uint32_t prune_batch_bytes() { return kPbBytes; }
uint32_t prune_kernel_smem_per_warp() { return 64 * (8 + 8 + 4) + kPbBytes; }

cudaError_t align_set_smem(uint32_t smem_bytes) {
    const int b = static_cast<int>(smem_bytes);
    cudaError_t e;
    if ((e = set_smem_variant<false, true, true>(b)) != cudaSuccess) return e;
    if ((e = set_smem_variant<false, true, false>(b)) != cudaSuccess) return e;
    if ((e = set_smem_variant<false, true, true, true>(b)) != cudaSuccess) return e;
    if ((e = set_smem_variant<false, true, true, false, true>(b)) != cudaSuccess) return e;
    if ((e = set_smem_variant<false, true, false, false, true>(b)) != cudaSuccess) return e;
    if ((e = set_smem_variant<false, true, false, true>(b)) != cudaSuccess) return e;
    if ((e = set_smem_variant<false, false, true>(b)) != cudaSuccess) return e;
    if ((e = set_smem_variant<false, false, false>(b)) != cudaSuccess) return e;
    if ((e = set_smem_variant<true, false, true>(b)) != cudaSuccess) return e;
    if ((e = set_smem_variant<true, false, false>(b)) != cudaSuccess) return e;
    return cudaFuncSetAttribute(lv_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
}

cudaError_t align_fast_occupancy(const AlignLaunch& a, int block, uint32_t smem_bytes, int* blocks_per_sm) {
    const bool reg = a.dl_max <= 15;
    if (a.prefetch)
        return reg ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, align_kernel<false, true, true>,
                                                                   block, smem_bytes)
                   : cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, align_kernel<false, true, false>,
                                                                   block, smem_bytes);
    return reg ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, align_kernel<false, false, true>, block,
                                                               smem_bytes)
               : cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, align_kernel<false, false, false>, block,
                                                               smem_bytes);
}

}  // namespace sab
