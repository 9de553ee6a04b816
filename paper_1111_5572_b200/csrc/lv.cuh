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
SA_DEV int lv_warp_reg(const uint4* R, int m, const uint4* W, uint32_t wofs, int w, int dl,
                       int lane, uint32_t& cells) {
    const int k = lane - dl;
    const bool mine = lane <= 2 * dl;
    int fr = kUnreach;
    for (int e = 0; e <= dl; ++e) {
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
template <bool kRegLV>
SA_DEV int lv_warp(const uint4* R, int m, const uint4* W, uint32_t wofs, int w, int dl, int* F,
                   int lane, uint32_t& cells, bool f16 = false) {
    if (kRegLV) return lv_warp_reg(R, m, W, wofs, w, dl, lane, cells);
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
    for (int t = 0; t < 2 * dl + 3; ++t) F[t * fs] = kU;
    const int off = dl + 1;
    for (int e = 0; e <= dl; ++e) {
        if (e > e_cap) return -2;
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

// standalone LV (lv_batch_kernel): any limit
SA_DEV int lv_warp_any(const uint4* R, int m, const uint4* W, uint32_t wofs, int w, int dl, int* F,
                       int lane, uint32_t& cells) {
    if (dl <= 15) return lv_warp_reg(R, m, W, wofs, w, dl, lane, cells);
    return lv_warp_smem(R, m, W, wofs, w, dl, F, lane, cells);
}

}  // namespace sab
