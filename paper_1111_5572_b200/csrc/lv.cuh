// lv.cuh -- warp-cooperative Landau-Vishkin bounded edit distance.
//
// bounded_distance (REF src/edit_distance.cpp:19-75): semi-global, read fully
// consumed, window start anchored, end free, unit costs, N never matches.
// Planes are uint4 {lo, hi, N, 0} blocks of 32 bases (common.cuh); R holds the
// read, W the window, window index j at plane bit wofs + j.  Either may live
// in shared or global memory (generic pointers).  Used by the aligner
// (align.cu) and the referee (referee.cu).
#pragma once
#include "common.cuh"

namespace sab {

#ifndef SA_LV_FULL
#define SA_LV_FULL
constexpr unsigned kLvFull = 0xffffffffu;
#endif


// Extend diagonal k from read index i while bases match (REF
// edit_distance.cpp:35-42; N never matches, :11-13).  R/W are shared-memory
// plane arrays; window index j lives at plane bit wofs + j.
SA_DEV int lv_slide(const uint4* R, const uint4* W, uint32_t wofs, int i, int k, int cap,
                    uint32_t& cells) {
    const int start = i;
    while (i < cap) {
        uint32_t rl, rh, rn, wl, wh, wn;
        extract32(R, static_cast<uint64_t>(i), rl, rh, rn);
        extract32(W, static_cast<uint64_t>(wofs + static_cast<uint32_t>(i + k)), wl, wh, wn);
        const uint32_t mism = (rl ^ wl) | (rh ^ wh) | rn | wn;
        if (mism == 0) {
            i += 32;
        } else {
            i += __ffs(mism) - 1;
            break;
        }
    }
    if (i > cap) i = cap;
    cells += static_cast<uint32_t>(i - start) + 1;
    return i;
}

// One LV iteration for diagonal k given the previous frontier values of
// k-1, k, k+1 (REF edit_distance.cpp:46-67).
SA_DEV int lv_step(int e, int k, int prev_km1, int prev_k, int prev_kp1, int m, int w,
                   const uint4* R, const uint4* W, uint32_t wofs, uint32_t& cells) {
    if (k > w) return kUnreach;  // whole diagonal outside the window (:47)
    int cand;
    if (e == 0) {
        cand = 0;
    } else {
        cand = prev_k + 1;                // substitution
        cand = max(cand, prev_kp1 + 1);   // extra read char
        cand = max(cand, prev_km1);       // extra window char
    }
    if (cand < max(0, -k)) return kUnreach;  // (:56-59)
    const int cap = min(m, w - k);
    cand = min(cand, cap);  // (:60)
    return lv_slide(R, W, wofs, cand, k, cap, cells);
}

// Register wavefront for d_limit <= 15: lane l owns diagonal k = l - d_limit.
// Iterations e_first..dl, from the frontier value `fr` of iteration e_first - 1.
SA_DEV int lv_warp_reg_from(int fr, int e_first, const uint4* R, int m, const uint4* W, uint32_t wofs, int w,
                            int dl, int lane, uint32_t& cells) {
    const int k = lane - dl;
    const bool mine = lane <= 2 * dl;
    for (int e = e_first; e <= dl; ++e) {
        int up = __shfl_down_sync(kLvFull, fr, 1);
        int dn = __shfl_up_sync(kLvFull, fr, 1);
        if (lane == 31) up = kUnreach;
        if (lane == 0) dn = kUnreach;
        const bool active = mine && k >= -e && k <= e;
        if (active) fr = lv_step(e, k, dn, fr, up, m, w, R, W, wofs, cells);
        if (__any_sync(kLvFull, active && fr == m)) return e;
    }
    return -1;
}

SA_DEV int lv_warp_reg(const uint4* R, int m, const uint4* W, uint32_t wofs, int w, int dl,
                       int lane, uint32_t& cells) {
    return lv_warp_reg_from(kUnreach, 0, R, m, W, wofs, w, dl, lane, cells);
}

// The register wavefront resumed from a serial one (lv_thread returned -2
// after iteration e0 < dl): F holds iteration e0's values of diagonals
// -e0..e0 in lv_thread's layout (16-bit entries, stride fs); the warp runs
// iterations e0 + 1..dl, lane per diagonal.  Same steps, same value.
SA_DEV int lv_warp_resume(const uint4* R, int m, const uint4* W, uint32_t wofs, int w, int dl,
                          const short* F, int fs, int e0, int lane, uint32_t& cells) {
    const int k = lane - dl;
    int fr = kUnreach;
    if (lane <= 2 * dl && k >= -e0 && k <= e0) {
        const int v = F[(k + dl + 1) * fs];
        if (v >= 0) fr = v;
    }
    return lv_warp_reg_from(fr, e0 + 1, R, m, W, wofs, w, dl, lane, cells);
}

// Shared-memory wavefront for any d_limit: F holds 2 * (2*dl + 3) entries of
// T.  T = short halves the frontier for reads < 32 k bases (every stored value
// is a read index <= m or "unreachable", kept as -32768: any negative value
// stays unreachable after +1, REF edit_distance.cpp:56-59).
template <typename T = int>
SA_DEV int lv_warp_smem(const uint4* R, int m, const uint4* W, uint32_t wofs, int w, int dl,
                        T* F, int lane, uint32_t& cells) {
    constexpr int kStoreUnreach = sizeof(T) == 2 ? -32768 : kUnreach;
    const int width = 2 * dl + 3;
    T* cur = F;
    T* nxt = F + width;
    for (int t = lane; t < 2 * width; t += 32) F[t] = static_cast<T>(kStoreUnreach);
    __syncwarp();
    const int off = dl + 1;
    for (int e = 0; e <= dl; ++e) {
        bool found = false;
        for (int k = -e + lane; k <= e; k += 32) {
            const int v = lv_step(e, k, cur[k - 1 + off], cur[k + off], cur[k + 1 + off], m, w, R,
                                  W, wofs, cells);
            nxt[k + off] = static_cast<T>(v < 0 ? kStoreUnreach : v);
            found |= (v == m);
        }
        __syncwarp();
        if (__any_sync(kLvFull, found)) return e;
        T* t = cur;
        cur = nxt;
        nxt = t;
    }
    return -1;
}

// kRegLV: every d_limit of the launch is <= 15 (register wavefront only);
// otherwise the shared-memory wavefront serves every limit.  One variant per
// kernel keeps the inlined code small.
SA_DEV int lv_bitpar_warp(const uint4* R, int nblk, int m, const uint4* W, uint32_t wofs, int w, int dl, int lane,
                          uint32_t& cells);
SA_DEV int lv_sys(const uint4* R, int nblk, int m, const uint4* W, uint32_t wofs, int w, int dl, int lane,
                  uint32_t& cells);

template <bool kRegLV, bool kSys = false>
SA_DEV int lv_warp(const uint4* R, int m, const uint4* W, uint32_t wofs, int w, int dl, int* F,
                   int lane, uint32_t& cells, bool f16 = false) {
    if (kRegLV) return lv_warp_reg(R, m, W, wofs, w, dl, lane, cells);
    if (kSys && SA_LV_LONG && dl >= SA_BITPAR_MIN_DL && dl <= kSysMaxDl)
        return lv_sys(R, (m + 31) / 32 + 1, m, W, wofs, w, dl, lane, cells);
    if (dl >= SA_BITPAR_MIN_DL && 2 * dl + 1 <= 2048)
        return lv_bitpar_warp(R, (m + 31) / 32 + 1, m, W, wofs, w, dl, lane, cells);
    if (f16) return lv_warp_smem(R, m, W, wofs, w, dl, reinterpret_cast<short*>(F), lane, cells);
    return lv_warp_smem(R, m, W, wofs, w, dl, F, lane, cells);
}

// Serial LV for one thread (d_limit <= 15): the frontier is 2*dl+3 16-bit
// entries at F[0], F[fs], F[2*fs], ... (shared memory, one column per thread)
// and is updated in place, diagonal by diagonal, carrying the old value of
// k-1 in a register.  Every diagonal of iteration e is stepped before the
// result is taken -- the steps, and so the dp_cells count, are exactly those
// of lv_warp_reg.  R and W are global plane arrays (read-only in this kernel).
// Returns -2 once e would exceed e_cap (< dl): the caller hands the read to
// the warp kernel, so one thread's long wavefront does not hold up its warp.
SA_DEV int lv_thread(const uint4* R, int m, const uint4* W, uint32_t wofs, int w, int dl, short* F, int fs,
                     uint32_t& cells, int e_cap) {
    constexpr short kU = -32768;  // unreachable: stays negative after +1 (REF edit_distance.cpp:56-59)
    const int off = dl + 1;
    for (int e = 0; e <= dl; ++e) {
        if (e > e_cap) return -2;
        // iteration e reads diagonals -e..e+1; -e, e and e+1 were never
        // written (iteration e-1 wrote -(e-1)..e-1), so only they are reset
        F[(off - e) * fs] = kU;
        F[(off + e) * fs] = kU;
        F[(off + e + 1) * fs] = kU;
        bool found = false;
        int left = kU;  // old value of diagonal k-1
        int cur = F[(off - e) * fs];
        for (int k = -e; k <= e; ++k) {
            const int right = F[(k + 1 + off) * fs];
            const int v = lv_step(e, k, left, cur, right, m, w, R, W, wofs, cells);
            left = cur;
            cur = right;
            F[(k + off) * fs] = static_cast<short>(v < 0 ? kU : v);
            found |= v == m;
        }
        if (found) return e;
    }
    return -1;
}


// Banded bit-parallel bounded edit distance for one thread (d_limit <= 15),
// same value as bounded_distance (REF src/edit_distance.cpp:19-75), computed
// with Myers' bit-vector column steps (Hyyrö's formulation, global variant)
// restricted to the diagonal band |j - i| <= dl, one 32-bit word per column:
// bit b of the column-j word is row i = j - dl + b.
//  * Cells outside the band are replaced by boundary values >= dl + 1 chosen
//    so every delta stays in {-1, 0, +1}: the row above the band's top enters
//    with horizontal delta +1 (the "| 1" shift-in), and the row that enters
//    at the bottom with vertical delta +1.  A path through a boundary cell
//    costs more than dl, so every value <= dl is exact, and every value > dl
//    stays > dl.
//  * Rows <= 0 are virtual never-matching rows with H[-r][j] = j + r (row 0 is
//    the anchored window start, D[0][j] = j); they satisfy the recurrence and
//    feed row 1 exactly as row 0 does.
//  * `top` tracks H at the band's top row along its diagonal (+1 unless the
//    top bit of D0 says the diagonal step is free); H[m][j] = top + the
//    vertical deltas from the top bit down to row m.
// Every thread with the same limit runs the same number of column steps, so
// a warp of reads stays converged (the serial wavefront diverged to ~3 active
// lanes per instruction).  dp_cells counts band cells (implementation-specific).
// R: read planes (nblk blocks; positions past the read carry N bits), W:
// genome planes with the window starting at base wofs, w bases long.
SA_DEV int lv_bitpar(const uint4* R, int nblk, int m, const uint4* W, uint32_t wofs, int w, int dl,
                     uint32_t& cells) {
    const int width = 2 * dl + 1;
    const uint32_t wmask = width >= 32 ? 0xffffffffu : ((1u << width) - 1u);
    uint32_t VP = wmask & ~((2u << dl) - 1u);  // column 0: rows 1..dl rise by 1
    uint32_t VN = (2u << dl) - 1u;             // rows -dl..0 fall by 1 (H[-r][0] = r)
    int top = dl;                              // H[-dl][0]
    int best = m <= dl ? m : 0x7fffffff;       // H[m][0] = m
    const int jend = min(w, m + dl);
    // read planes for positions q .. q+31, q = j - 1 - dl (blocks qb, qb + 1)
    auto blk = [&](int b) -> uint4 {
        return (b < 0 || b >= nblk) ? make_uint4(0u, 0u, 0xffffffffu, 0u) : R[b];
    };
    int q = -dl;  // j = 1
    int qb = q >> 5;
    uint4 A = blk(qb), B = blk(qb + 1);
    uint32_t gp = wofs;  // window base j - 1
    uint4 G = W[gp >> 5];
    for (int j = 1; j <= jend; ++j) {
        if ((q >> 5) != qb) {
            ++qb;
            A = B;
            B = blk(qb + 1);
        }
        if ((gp & 31u) == 0u && j > 1) G = W[gp >> 5];
        const uint32_t sh = static_cast<uint32_t>(q & 31);
        const uint32_t rl = __funnelshift_r(A.x, B.x, sh), rh = __funnelshift_r(A.y, B.y, sh);
        const uint32_t rn = __funnelshift_r(A.z, B.z, sh);
        const uint32_t gb = gp & 31u;
        const uint32_t tl = 0u - ((G.x >> gb) & 1u), th = 0u - ((G.y >> gb) & 1u), tn = 0u - ((G.z >> gb) & 1u);
        const uint32_t eq = ~((rl ^ tl) | (rh ^ th) | rn | tn);  // N never matches (REF edit_distance.cpp:11-13)
        VP = (VP >> 1) | (1u << (width - 1));
        VN >>= 1;
        const uint32_t D0 = ((((eq & VP) + VP) ^ VP) | eq | VN);
        const uint32_t HP = VN | ~(D0 | VP);
        const uint32_t HN = VP & D0;
        top += (D0 & 1u) ^ 1u;
        const uint32_t X = (HP << 1) | 1u;
        VN = X & D0 & wmask;
        VP = ((HN << 1) | ~(X | D0)) & wmask;
        const int bm = m - j + dl;  // bit of row m (>= 0 since j <= m + dl)
        if (bm < width) {
            const uint32_t mk = (bm >= 31 ? 0xffffffffu : ((2u << bm) - 1u)) & ~1u;
            best = min(best, top + __popc(VP & mk) - __popc(VN & mk));
        }
        ++q;
        ++gp;
    }
    cells += static_cast<uint32_t>(jend > 0 ? jend : 0) * static_cast<uint32_t>(width);
    return best <= dl ? best : -1;
}

// ---------------------------------------------------------------- mask LV
// Segmented register wavefront with precomputed mismatch masks, for reads of
// at most 128 bases and d_limit <= 15 (same values as bounded_distance, REF
// src/edit_distance.cpp:19-75).  The warp is cut into segments of
// 2*dl + 1 lanes, one (read orientation, window) job per segment, lane
// k + dl of a segment owning diagonal k.  Before the wavefront each lane
// builds the 128-bit mismatch mask of its diagonal -- bit i set when read
// base i differs from window base i + k or either is N (REF :11-13), and
// every bit at or past cap = min(m, w - k) set -- from a handful of
// independent loads issued together, so the slides are bit scans in
// registers instead of a chain of dependent memory reads.  The recurrence,
// guards and clamps are lv_step's exactly.
constexpr int kMaskMaxLen = 128;

// First set bit at or after i (0 <= i <= 128) of a 128-bit mask; 128 if none.
SA_DEV int mask_next(const uint32_t (&M)[4], int i) {
    const int q = i >> 5;
    const uint32_t lc = ~0u << (i & 31);
    const uint32_t t0 = q == 0 ? (M[0] & lc) : 0u;
    const uint32_t t1 = q == 1 ? (M[1] & lc) : (q < 1 ? M[1] : 0u);
    const uint32_t t2 = q == 2 ? (M[2] & lc) : (q < 2 ? M[2] : 0u);
    const uint32_t t3 = q == 3 ? (M[3] & lc) : (q < 3 ? M[3] : 0u);
    if (t0) return __ffs(t0) - 1;
    if (t1) return 31 + __ffs(t1);
    if (t2) return 63 + __ffs(t2);
    if (t3) return 95 + __ffs(t3);
    return 128;
}

// 32 genome bases at signed position p (bases before 0 or past the padded
// planes read as N).  nbg = ceil(glen / 32): planes[0 .. nbg + 1] exist.
SA_DEV void extract32_any(const uint4* planes, uint64_t nbg, int64_t p, uint32_t& lo, uint32_t& hi, uint32_t& n) {
    if (p < 0) {
        const int sft = static_cast<int>(-p);  // < 32
        extract32_ldg(planes, 0, lo, hi, n);
        lo <<= sft;
        hi <<= sft;
        n = (n << sft) | ((1u << sft) - 1u);
    } else if ((static_cast<uint64_t>(p) >> 5) > nbg) {
        lo = hi = 0;
        n = 0xffffffffu;
    } else {
        extract32_ldg(planes, static_cast<uint64_t>(p), lo, hi, n);
    }
}

// Segment jobs: this lane's segment reads R (m bases) against the genome
// window starting at `anchor`, w bases long; live = the segment has a job.
// Returns, in every lane of a live segment, its distance (<= dl) or -1.
SA_DEV int lv_seg(const uint4* R, int m, const uint4* G, uint64_t nbg, uint64_t anchor, int w, bool live, int dl,
                  int lane, uint32_t& cells) {
    const int wd = 2 * dl + 1;
    const int seg = lane / wd;
    const int k = lane - seg * wd - dl;
    const bool in = live && seg < 32 / wd;
    const int cap = min(m, w - k);
    uint32_t M[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        M[q] = 0xffffffffu;
        if (in && 32 * q < m && 32 * q < cap) {
            const uint4 r = R[q];
            uint32_t wl, wh, wn;
            extract32_any(G, nbg, static_cast<int64_t>(anchor) + k + 32 * q, wl, wh, wn);
            M[q] = (r.x ^ wl) | (r.y ^ wh) | r.z | wn;
        }
        const int b0 = 32 * q;
        if (cap <= b0) M[q] = 0xffffffffu;
        else if (cap < b0 + 32) M[q] |= ~0u << (cap - b0);
    }
    const uint32_t segmask = in ? (((wd >= 32) ? 0xffffffffu : ((1u << wd) - 1u)) << (seg * wd)) : 0u;
    int fr = kUnreach, res = -1;
    bool done = !in;
    for (int e = 0; e <= dl; ++e) {
        int up = __shfl_down_sync(kLvFull, fr, 1);
        int dn = __shfl_up_sync(kLvFull, fr, 1);
        if (k == dl) up = kUnreach;
        if (k == -dl) dn = kUnreach;
        const bool active = !done && k >= -e && k <= e;
        if (active) {
            if (k > w) {
                fr = kUnreach;  // whole diagonal outside the window (REF :47)
            } else {
                int cand = e == 0 ? 0 : max(max(fr + 1, up + 1), dn);
                if (cand < max(0, -k)) {
                    fr = kUnreach;  // (REF :56-59)
                } else {
                    cand = min(cand, cap);  // (REF :60)
                    const int i = min(mask_next(M, cand), cap);
                    cells += static_cast<uint32_t>(i - cand) + 1;
                    fr = i;
                }
            }
        }
        const uint32_t hit = __ballot_sync(kLvFull, active && fr == m);
        if (!done && (hit & segmask)) {
            done = true;
            res = e;
        }
        if (__all_sync(kLvFull, done)) break;
    }
    return res;
}

// ---------------------------------------------------------------- warp bit-parallel LV
// Banded bit-parallel bounded edit distance for large limits (long reads),
// warp-cooperative: lv_bitpar's column recurrence (Myers/Hyyro, band of
// W = 2 dl + 1 rows, boundary cells >= dl + 1 so every value <= dl is exact
// and every value > dl stays > dl) with the band spread over the warp, lane l
// holding band bits 64 l .. 64 l + 63 (W <= 2048, dl <= 1023).  Per column:
// the eq word from the read planes, the band shifted down one row (bit 0 of
// the next lane), the addition with its carry scanned across lanes
// (generate/propagate, 5 shuffles), the HP/HN shift up (bit 63 of the previous
// lane).  Same value as bounded_distance (REF src/edit_distance.cpp:19-75).
//
// It also stops early: every 64 columns the band's minimum H (top plus the
// least prefix of the vertical deltas, scanned across lanes) is taken; once
// it exceeds dl no later cell -- every path to row m runs through this column's
// band, and DP values never fall along a path -- can be <= dl.  The
// wavefront LV must reach iteration dl + 1 to say "more than dl"
// (sum over e of 2e + 1 steps); for a long diverged read this stops where the
// band's minimum crosses dl.
SA_DEV uint64_t shfl64_lv(uint64_t v, int src) {
    const uint32_t lo = __shfl_sync(kLvFull, static_cast<uint32_t>(v), src);
    const uint32_t hi = __shfl_sync(kLvFull, static_cast<uint32_t>(v >> 32), src);
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

// 64 read bases from position q (may be negative or past the read: N) of
// planes R (nblk blocks).
SA_DEV void read64(const uint4* R, int nblk, int q, uint64_t& l, uint64_t& h, uint64_t& n) {
    auto blk = [&](int b) -> uint4 { return (b < 0 || b >= nblk) ? make_uint4(0u, 0u, 0xffffffffu, 0u) : R[b]; };
    const int b = q >> 5;  // arithmetic shift: floor
    const uint32_t sh = static_cast<uint32_t>(q & 31);
    const uint4 A = blk(b), B = blk(b + 1), C = blk(b + 2);
    const uint32_t l0 = __funnelshift_r(A.x, B.x, sh), l1 = __funnelshift_r(B.x, C.x, sh);
    const uint32_t h0 = __funnelshift_r(A.y, B.y, sh), h1 = __funnelshift_r(B.y, C.y, sh);
    const uint32_t n0 = __funnelshift_r(A.z, B.z, sh), n1 = __funnelshift_r(B.z, C.z, sh);
    l = (static_cast<uint64_t>(l1) << 32) | l0;
    h = (static_cast<uint64_t>(h1) << 32) | h0;
    n = (static_cast<uint64_t>(n1) << 32) | n0;
}

SA_DEV int lv_bitpar_warp(const uint4* R, int nblk, int m, const uint4* W, uint32_t wofs, int w, int dl, int lane,
                          uint32_t& cells) {
    const int width = 2 * dl + 1;
    const int b0 = 64 * lane;  // this lane's first band bit
    auto range = [&](int lo, int hi) -> uint64_t {  // bits [lo, hi] of the band in this lane's word
        const int a = max(lo, b0), b = min(hi, b0 + 63);
        if (a > b) return 0ull;
        const int len = b - a + 1;
        return (len == 64 ? ~0ull : ((1ull << len) - 1ull)) << (a - b0);
    };
    const uint64_t wmask = range(0, width - 1);
    const bool top_lane_has = (width - 1) >= b0 && (width - 1) <= b0 + 63;
    const uint64_t inject = top_lane_has ? (1ull << ((width - 1) - b0)) : 0ull;
    uint64_t VP = range(dl + 1, 2 * dl);  // column 0: rows 1..dl rise by 1
    uint64_t VN = range(0, dl);           // rows -dl..0 fall by 1 (H[-r][0] = r)
    int top = dl;                          // H[-dl][0]
    int best = m <= dl ? m : 0x7fffffff;  // H[m][0] = m
    const int jend = min(w, m + dl);
    int j = 1;
    for (; j <= jend; ++j) {
        const int q = j - 1 - dl + b0;  // read position of this lane's band bit 0
        uint64_t rl, rh, rn;
        read64(R, nblk, q, rl, rh, rn);
        const uint32_t gpos = wofs + static_cast<uint32_t>(j - 1);
        const uint4 G = W[gpos >> 5];
        const uint32_t gb = gpos & 31u;
        const uint64_t tl = 0ull - ((G.x >> gb) & 1u), th = 0ull - ((G.y >> gb) & 1u), tn = 0ull - ((G.z >> gb) & 1u);
        const uint64_t eq = ~((rl ^ tl) | (rh ^ th) | rn | tn) & wmask;  // N never matches (REF edit_distance.cpp:11-13)
        // band down one row
        const uint64_t vp_up = shfl64_lv(VP, (lane + 1) & 31), vn_up = shfl64_lv(VN, (lane + 1) & 31);
        VP = ((VP >> 1) | (lane < 31 ? (vp_up << 63) : 0ull)) & wmask;
        VN = ((VN >> 1) | (lane < 31 ? (vn_up << 63) : 0ull)) & wmask;
        VP |= inject;
        // (eq & VP) + VP with the carry across lanes
        const uint64_t xa = eq & VP;
        uint64_t sum = xa + VP;
        uint32_t g = sum < xa ? 1u : 0u;              // carry out with no carry in
        uint32_t pr = sum == ~0ull ? 1u : 0u;         // a carry in would pass through
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {  // inclusive scan of (g, p): carry out of lanes <= this one
            const uint32_t g2 = __shfl_up_sync(kLvFull, g, o), p2 = __shfl_up_sync(kLvFull, pr, o);
            if (lane >= o) {
                g = g | (pr & g2);
                pr = pr & p2;
            }
        }
        const uint32_t cin = __shfl_up_sync(kLvFull, g, 1);  // every lane takes part
        sum += lane > 0 ? cin : 0u;
        const uint64_t D0 = ((sum ^ VP) | eq | VN);
        const uint64_t HP = VN | ~(D0 | VP);
        const uint64_t HN = VP & D0;
        top += static_cast<int>((__shfl_sync(kLvFull, static_cast<uint32_t>(D0), 0) & 1u) ^ 1u);
        const uint64_t hp_lo = shfl64_lv(HP, (lane + 31) & 31), hn_lo = shfl64_lv(HN, (lane + 31) & 31);
        const uint64_t X = (HP << 1) | (lane > 0 ? (hp_lo >> 63) : 1ull);
        const uint64_t HNs = (HN << 1) | (lane > 0 ? (hn_lo >> 63) : 0ull);
        VN = X & D0 & wmask;
        VP = (HNs | ~(X | D0)) & wmask;
        const int bm = m - j + dl;  // band bit of row m
        if (bm < width) {
            const uint64_t mk = range(1, bm);
            const int v = __reduce_add_sync(kLvFull, static_cast<uint32_t>(__popcll(VP & mk))) -
                          __reduce_add_sync(kLvFull, static_cast<uint32_t>(__popcll(VN & mk)));
            best = min(best, top + v);
        }
        if ((j & 63) == 0 && best > dl) {  // the band's minimum: past dl, nothing later can reach row m within dl
            const uint64_t vp = VP & ~range(0, 0), vn = VN & ~range(0, 0);  // deltas of rows 1..
            int run = 0, lmin = 0x7fffffff;
            for (int t = 0; t < 64; ++t) {
                run += static_cast<int>((vp >> t) & 1ull) - static_cast<int>((vn >> t) & 1ull);
                lmin = min(lmin, run);
            }
            // exclusive prefix of the lanes' sums
            int pre = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t2 = __shfl_up_sync(kLvFull, pre, o);
                if (lane >= o) pre += t2;
            }
            pre -= run;
            const int mn = static_cast<int>(__reduce_min_sync(kLvFull, static_cast<uint32_t>(min(0, pre + lmin) + (1 << 20))))
                           - (1 << 20);
            if (top + mn > dl) {
                ++j;
                break;
            }
        }
    }
    cells += static_cast<uint32_t>(j - 1 > 0 ? j - 1 : 0) * static_cast<uint32_t>(width);
    return best <= dl ? best : -1;
}

// ---------------------------------------------------------------- systolic LV
// Banded bit-parallel bounded edit distance for large limits (long reads),
// lane per row block with the blocks skewed in time (a systolic array):
// the same value as bounded_distance (REF src/edit_distance.cpp:19-75), i.e.
// min over window prefixes j <= w of the global edit distance D[m][j] when it
// is <= dl, as lv_bitpar computes it.
//
// Rows (read bases) are cut into B = ceil(m / 64) blocks of 64 that END at
// row m (block b: rows r0(b) = m - 64 (B - b) + 1 .. r0(b) + 63; rows <= 0
// are virtual never-matching rows with D[-r][j] = j + r, which satisfy the
// recurrence and feed row 1 as row 0 does -- see lv_bitpar).  Each block
// keeps Myers/Hyyro vertical deltas (Pv, Mv) and D at its last row (sc);
// column j advances it with one word step given the horizontal delta
// entering at its top (hin, from the block above).  Block b runs columns
// 2p - 1 and 2p at time t = p + b, on lane b mod 32: the block above finished
// them at t - 1, so one shuffle per step carries (both hin, sc) down the warp
// and no carry has to cross lanes inside a step (lv_bitpar_warp's 5-step
// carry scan); two columns per step halve the per-step bookkeeping.
//
// Band: block b runs only the columns [r0 - dl, r0 + 63 + dl] (cells with
// |row - col| <= dl).  Outside them, values are replaced by upper bounds: the
// block above a block's first column holds "+1 per row" (Pv = ~0), and a
// block whose upper neighbour has left the band sees hin = +1.  Computed
// values are >= the true ones everywhere and equal on every cell whose true
// value is <= dl (such a cell's optimal path stays in the band), so the
// minimum over row m is exact whenever it is <= dl.  Every 64 steps the warp
// stops once every running block's lower bound (sc - popcount(Pv)) exceeds
// min(dl, best - 1) + 2: no later cell can be <= dl or beat the best found
// (the two-column skew between neighbours costs the + 2).
// dl <= kSysMaxDl (960, common.cuh) keeps one running block per lane (block
// b + 32 starts after b ends).

SA_DEV int lv_sys(const uint4* R, int nblk, int m, const uint4* W, uint32_t wofs, int w, int dl, int lane,
                  uint32_t& cells) {
    const int B = (m + 63) >> 6;
    const int jend = min(w, m + dl);
    int best = m <= dl ? m : 0x3fffffff;  // D[m][0] = m
    if (jend >= 1 && B > 0) {
        constexpr int kNever = 0x3fffffff;
        // two columns per step: block b runs columns 2p - 1, 2p at time p + b
        const int tmax = ((jend + 1) >> 1) + B - 1;
        int b = lane - 32;                    // current block (loaded at t == tsw)
        int tsw = lane < B ? 1 : kNever;      // time of the next block switch
        int ts = kNever, te = -1;             // running steps [ts, te] of the current block
        int js = 1, je = 0, ae = -kNever;     // its columns, and the block above's last column
        uint64_t Pv = 0, Mv = 0, q0 = 0, q1 = 0, q2 = 0, q3 = 0;
        int sc = 0;
        bool fresh = false;
        uint32_t gp = 0, gx = 0, gy = 0, gz = 0;
        int pub = 0;  // published each step: (sc << 4) | (hout(2p - 1) + 1) << 2 | (hout(2p) + 1)
        uint32_t cols = 0;
        const bool last_lane_block = ((B - 1) & 31) == lane;
        // one column of this lane's block: Myers/Hyyro word step, hin entering at the top
        auto column = [&](int hin) -> int {
            if ((gp & 31u) == 0u) {
                const uint4 G = W[gp >> 5];
                gx = G.x;
                gy = G.y;
                gz = G.z;
            }
            const uint64_t eqlo = (gx & 1u) ? q1 : q0, eqhi = (gx & 1u) ? q3 : q2;
            const uint64_t Eq0 = (gz & 1u) ? 0ull : ((gy & 1u) ? eqhi : eqlo);  // N never matches
            gx >>= 1;
            gy >>= 1;
            gz >>= 1;
            ++gp;
            const uint64_t hneg = hin < 0 ? 1ull : 0ull;
            const uint64_t Xv = Eq0 | Mv;
            const uint64_t Eq = Eq0 | hneg;
            const uint64_t Xh = (((Eq & Pv) + Pv) ^ Pv) | Eq;
            uint64_t Ph = Mv | ~(Xh | Pv);
            uint64_t Mh = Pv & Xh;
            const int hout = static_cast<int>(Ph >> 63) - static_cast<int>(Mh >> 63);
            Ph = (Ph << 1) | (hin > 0 ? 1ull : 0ull);
            Mh = (Mh << 1) | hneg;
            Pv = Mh | ~(Xv | Ph);
            Mv = Ph & Xv;
            ++cols;
            return hout;
        };
        bool act = false;
        for (int t = 1; t <= tmax; ++t) {
            const int rcv = __shfl_sync(kLvFull, pub, (lane + 31) & 31);
            if (t == tsw) {  // this lane's next block
                b += 32;
                const int r0 = m - 64 * (B - b) + 1;
                js = max(1, r0 - dl);
                je = min(jend, r0 + 63 + dl);
                ts = ((js + 1) >> 1) + b;
                te = ((je + 1) >> 1) + b;
                tsw = b + 32 < B ? te + 1 : kNever;
                ae = b > 0 ? min(jend, r0 - 1 + dl) : -kNever;
                uint64_t l, h, n;
                read64(R, nblk, r0 - 1, l, h, n);  // rows r0 .. r0 + 63 = read bases r0 - 1 ..
                q0 = ~(l | h | n);                 // eq masks per genome base (lo, hi) = (0,0) (1,0) (0,1) (1,1)
                q1 = l & ~h & ~n;
                q2 = ~l & h & ~n;
                q3 = l & h & ~n;
                if (js == 1) {  // exact column 0: D[row][0] = |row|
                    const int t1 = 1 - r0;  // first real row's bit
                    Pv = t1 <= 0 ? ~0ull : (t1 >= 64 ? 0ull : (~0ull << t1));
                    Mv = ~Pv;
                    sc = abs(r0 + 63);
                    fresh = false;
                } else {  // "+1 per row" below the block above (an upper bound, outside the band)
                    Pv = ~0ull;
                    Mv = 0ull;
                    fresh = true;
                }
                gp = wofs + static_cast<uint32_t>(js - 1);  // window base of column js
                const uint4 G = W[gp >> 5];
                gx = G.x >> (gp & 31u);
                gy = G.y >> (gp & 31u);
                gz = G.z >> (gp & 31u);
            }
            act = t >= ts && t <= te;
            if (act) {
                const int j2 = 2 * (t - b), j1 = j2 - 1;
                const int h1a = ((rcv >> 2) & 3) - 1, h2a = (rcv & 3) - 1, sce = rcv >> 4;
                const int hin1 = j1 <= ae ? h1a : 1;  // the block above left the band: +1
                const int hin2 = j2 <= ae ? h2a : 1;
                int ho1 = 0, ho2 = 0;
                const bool last = last_lane_block && b == B - 1;
                if (j1 >= js) {
                    // a new block's bottom before its first column: the block above's D
                    // there (its D at j1 is its published sc less its hout at j2) + 64
                    if (fresh) sc = sce - (j2 <= ae ? h2a : 0) - hin1 + 64;
                    fresh = false;
                    ho1 = column(hin1);
                    sc += ho1;
                    if (last) best = min(best, sc);  // D[m][j1]
                }
                if (j2 <= je) {
                    if (fresh) sc = sce - hin2 + 64;
                    fresh = false;
                    ho2 = column(hin2);
                    sc += ho2;
                    if (last) best = min(best, sc);  // D[m][j2]
                }
                pub = (sc << 4) | ((ho1 + 1) << 2) | (ho2 + 1);
            }
            if ((t & 63) == 0) {
                // neighbours are one step (two columns) apart: future cells stay
                // above min(dl, best - 1) once every running block's bound exceeds it by 2
                const int bw = static_cast<int>(__reduce_min_sync(kLvFull, static_cast<uint32_t>(best)));
                const int thr = min(dl + 2, bw + 1);
                const bool done = !act || sc - __popcll(Pv) > thr;
                if (__all_sync(kLvFull, done)) break;
            }
        }
        cells += cols * 64u;
    }
    best = static_cast<int>(__reduce_min_sync(kLvFull, static_cast<uint32_t>(best)));
    return best <= dl ? best : -1;
}

// ---------------------------------------------------------------- q-gram filter
// An exact pre-test that proves bounded_distance(read, window, dl) > dl
// without running the LV (the result is then -1, as the LV's would be).
// q-gram lemma: an alignment with at most dl edits leaves at least
// (m - q + 1) - dl q of the read's q-grams (by position) untouched -- a
// substitution or an inserted read base touches the q q-grams covering it, a
// deleted window base the q - 1 spanning its gap -- and an untouched q-gram
// occurs in the aligned window prefix, within dl of its own position (the
// alignment never leaves the band |row - col| <= dl).  A q-gram holding N is
// never untouched (N never matches, REF edit_distance.cpp:11-13).  So the
// read is cut into pieces of kQfPiece q-gram starts; for each piece the set of
// window q-grams in the piece's band [a - dl, b - 1 + dl] goes into a
// 4^kQfQ-bit bitmap (bm, 512 B of the warp's shared memory) and the piece's
// read q-grams found in it are counted; fewer than the bound in total proves
// the distance > dl.  Stops as soon as the bound is reached (run the LV) or
// cannot be reached any more (reject).  C3 (1 kbp reads, dl 83): 98% of its
// LVs fail, and this rejects ~83% of those (measured on a CPU model of the
// call sequence).
constexpr int kQfQ = 6;        // q
constexpr int kQfPiece = 128;  // read q-gram starts per piece

SA_DEV bool qgram_reject(const uint4* R, int m, const uint4* W, uint32_t wofs, int w, int dl, uint32_t* bm,
                         int lane) {
    const int nq = m - kQfQ + 1;
    const int thr = nq - dl * kQfQ;
    if (thr <= 0) return false;
    constexpr uint32_t kMask = (1u << kQfQ) - 1u;
    int total = 0;
    for (int a0 = 0; a0 < nq; a0 += kQfPiece) {
        const int b0 = min(nq, a0 + kQfPiece);
        const int lo = max(0, a0 - dl), hi = min(w - kQfQ, b0 - 1 + dl);  // window q-gram starts
        for (int t = lane; t < (1 << (2 * kQfQ)) / 32; t += 32) bm[t] = 0u;
        __syncwarp();
        for (int j = lo + lane; j <= hi; j += 32) {
            uint32_t l, h, n;
            extract32(W, static_cast<uint64_t>(wofs) + static_cast<uint32_t>(j), l, h, n);
            if ((n & kMask) == 0u) {
                const uint32_t v = (l & kMask) | ((h & kMask) << kQfQ);
                atomicOr(bm + (v >> 5), 1u << (v & 31u));
            }
        }
        __syncwarp();
        int c = 0;
        for (int i = a0 + lane; i < b0; i += 32) {
            uint32_t l, h, n;
            extract32(R, static_cast<uint64_t>(i), l, h, n);
            if ((n & kMask) == 0u) {
                const uint32_t v = (l & kMask) | ((h & kMask) << kQfQ);
                c += static_cast<int>((bm[v >> 5] >> (v & 31u)) & 1u);
            }
        }
        total += static_cast<int>(__reduce_add_sync(kLvFull, static_cast<uint32_t>(c)));
        __syncwarp();
        if (total >= thr) return false;          // the bound can be met: run the LV
        if (total + (nq - b0) < thr) return true;  // not even with every later q-gram
    }
    return total < thr;
}

// standalone LV (lv_batch_kernel): any limit; bitpar_min = the limit from
// which the warp bit-parallel LV serves (test hook: lower it to cover it)
SA_DEV int lv_warp_any(const uint4* R, int m, const uint4* W, uint32_t wofs, int w, int dl, int* F,
                       int lane, uint32_t& cells, int bitpar_min = SA_BITPAR_MIN_DL, bool long_bitpar = !SA_LV_LONG) {
    if (dl <= 15) return lv_warp_reg(R, m, W, wofs, w, dl, lane, cells);
    if (!long_bitpar && dl >= bitpar_min && dl <= kSysMaxDl) return lv_sys(R, (m + 31) / 32 + 1, m, W, wofs, w, dl, lane, cells);
    if (dl >= bitpar_min && 2 * dl + 1 <= 2048)
        return lv_bitpar_warp(R, (m + 31) / 32 + 1, m, W, wofs, w, dl, lane, cells);
    return lv_warp_smem(R, m, W, wofs, w, dl, F, lane, cells);
}

}  // namespace sab
