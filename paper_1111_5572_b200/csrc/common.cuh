// common.cuh -- device-side vocabulary shared by the index build, the lookup
// kernel, the LV kernel and the fused per-read align kernel.
//
// Genome in HBM ("bit planes"): one uint4 per 32-base block b,
//   .x = low code bits, .y = high code bits, .z = N bits, .w = 0,
// bit j of each plane = genome base 32*b + j.  Codes follow the reference
// (A=0 C=1 G=2 T=3, REF include/seedaln/genome.hpp:13); N positions carry the
// N bit (REF genome.hpp:50-54).  Blocks past the genome end are all-N, and two
// padding blocks follow the last one so a 32-base window read at any valid
// position (which touches blocks b and b+1) never leaves the allocation.
// Comparing 32 bases is (lo^lo')|(hi^hi')|n|n' on 32-bit words; the first
// mismatch is __ffs of that.
//
// Seed index ("slots"): open-addressing table keyed by the canonical seed
// key min(key, rc(key)).  Slot = {u64 key, u32 payload, u32 meta}; empty key
// = ~0 (never canonical: all-T has rc all-A = 0).  meta bits 0..30 = number
// of genome windows whose key is canon or rc(canon); bit 31 = strand flag of
// a singleton.  n == 1: payload = the window position (inline).  n > 1:
// payload = offset into the position pool, pool[payload] = n_fwd (windows
// equal to canon), then n positions: the n_fwd canon-strand windows, then the
// rc-strand ones, each group ascending.  One probe answers both of the
// reference's binary searches (REF src/seed_index.cpp:128-143).
#pragma once
#include <cstdint>

#define SA_DEV __device__ __forceinline__

namespace sab {

// Long-read LV (lv.cuh): limits from SA_BITPAR_MIN_DL up to kSysMaxDl use the
// systolic bit-parallel lv_sys (SA_LV_LONG 1) or lv_bitpar_warp (0, and above
// kSysMaxDl up to 1023); below, the LV wavefronts.
#ifndef SA_BITPAR_MIN_DL
#define SA_BITPAR_MIN_DL 256
#endif
#ifndef SA_LV_LONG
#define SA_LV_LONG 1
#endif
constexpr int kSysMaxDl = 960;

constexpr uint64_t kEmptyKey = ~0ull;
constexpr int kInfDistance = 0x7fffffff / 4;  // REF include/seedaln/aligner.hpp:15
constexpr int kGapCap = 1000;                 // REF aligner.hpp:34
constexpr int kUnreach = -(1 << 30);          // LV "unreachable" (REF edit_distance.cpp:15)

struct Slot {
    unsigned long long key;
    unsigned int payload;
    unsigned int meta;
};

// 32 -> 64 bit spread: bit j -> bit 2j.
SA_DEV uint64_t spread32(uint32_t v) {
    uint64_t x = v;
    x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
    x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
    x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    return x;
}

SA_DEV uint32_t seed_mask32(int s) { return s >= 32 ? 0xffffffffu : ((1u << s) - 1u); }

// Seed keys in "planar" form: key = (hi bits << s) | lo bits of the s-base
// string (bit j = base j).  This is a bijection of the reference's packed key
// (REF src/seed_index.cpp:51-60, first base in the high bits), so equality,
// palindromes and the canonical pair {q, rc(q)} are the same; only the choice
// of representative (the smaller planar key) differs, and build and probe use
// the same rule.  It costs a few ALU ops instead of 2-bit interleaving.
SA_DEV uint64_t planar_key(uint32_t lo, uint32_t hi, int s) {
    const uint32_t m = seed_mask32(s);
    return (static_cast<uint64_t>(hi & m) << s) | (lo & m);
}

// Planar key of the reverse complement (REF src/seed_index.cpp:62-70): the
// complement flips both code bits (A<->T, C<->G); reversal is __brev.
SA_DEV uint64_t planar_rc_key(uint32_t lo, uint32_t hi, int s) {
    const uint32_t rl = __brev(~lo) >> (32 - s);
    const uint32_t rh = __brev(~hi) >> (32 - s);
    return (static_cast<uint64_t>(rh) << s) | rl;
}

// Reference packed key (first base high) of the same string, for tests.
SA_DEV uint64_t packed_key(uint32_t lo, uint32_t hi, int s) {
    uint64_t f = spread32(__brev(lo)) | (spread32(__brev(hi)) << 1);
    return f >> (64 - 2 * s);
}

SA_DEV uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

SA_DEV uint64_t home_slot(uint64_t canon, uint64_t n_slots) { return __umul64hi(mix64(canon), n_slots); }

// 32 bases starting at absolute base position p of a plane array.
SA_DEV void extract32(const uint4* planes, uint64_t p, uint32_t& lo, uint32_t& hi, uint32_t& n) {
    const uint64_t b = p >> 5;
    const uint32_t sh = static_cast<uint32_t>(p & 31);
    const uint4 a = planes[b];
    const uint4 c = planes[b + 1];
    lo = __funnelshift_r(a.x, c.x, sh);
    hi = __funnelshift_r(a.y, c.y, sh);
    n = __funnelshift_r(a.z, c.z, sh);
}

// Same, reading through the read-only path (global genome).
SA_DEV void extract32_ldg(const uint4* planes, uint64_t p, uint32_t& lo, uint32_t& hi, uint32_t& n) {
    const uint64_t b = p >> 5;
    const uint32_t sh = static_cast<uint32_t>(p & 31);
    const uint4 a = __ldg(planes + b);
    const uint4 c = __ldg(planes + b + 1);
    lo = __funnelshift_r(a.x, c.x, sh);
    hi = __funnelshift_r(a.y, c.y, sh);
    n = __funnelshift_r(a.z, c.z, sh);
}

// Reference base code of an ASCII read character for the aligner:
// 0..3 = ACGT, 4 = 'N', 5 = anything else (reverse_complement rejects it,
// REF src/genome.cpp:182-200).
SA_DEV int read_code(unsigned char ch) {
    switch (ch) {
        case 'A': return 0;
        case 'C': return 1;
        case 'G': return 2;
        case 'T': return 3;
        case 'N': return 4;
        default: return 5;
    }
}

// Probe the table for a canonical key.  Returns false on a miss.
SA_DEV bool probe_from(const Slot* __restrict__ table, uint64_t n_slots, uint64_t canon, uint64_t h,
                       unsigned int& payload, unsigned int& meta) {
    const ulonglong2* t = reinterpret_cast<const ulonglong2*>(table);
    for (;;) {
        ulonglong2 v = __ldg(t + h);
        if (v.x == canon) {
            payload = static_cast<unsigned int>(v.y);
            meta = static_cast<unsigned int>(v.y >> 32);
            return true;
        }
        if (v.x == kEmptyKey) return false;
        h = (h + 1 == n_slots) ? 0 : h + 1;
    }
}

SA_DEV bool probe_slot(const Slot* __restrict__ table, uint64_t n_slots, uint64_t canon,
                       unsigned int& payload, unsigned int& meta) {
    return probe_from(table, n_slots, canon, home_slot(canon, n_slots), payload, meta);
}

}  // namespace sab
