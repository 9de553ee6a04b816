/*
 * snap_oracle.c -- TEST INFRASTRUCTURE ONLY (see snap_oracle.h).
 *
 * Plain-C restatement of the reference aligner hot path.  Every function
 * cites the reference lines it follows (REF = /root/reference/proj).  It is
 * deliberately literal -- sorted CSR index, binary-search lookups, a
 * candidate vector plus hash map, the serial LV wavefront -- so that it reads
 * against the reference line by line.  It is the checker, never the product.
 */
#define _GNU_SOURCE
#include "snap_oracle.h"

#include <limits.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>

#define K_INF_DISTANCE (INT_MAX / 4) /* REF aligner.hpp:15 */
#define K_GAP_CAP 1000               /* REF aligner.hpp:34 */

/* ------------------------------------------------------------ genome */

/* REF src/genome.cpp:27-41 char_to_base: A/C/G/T any case, IUPAC -> N. */
/* 0..3 ACGT (any case), 4 the IUPAC N class, -1 otherwise (REF genome.cpp
 * char_to_base); a table, since random bases defeat a branchy switch */
static const signed char g_code[256] = {
    [0 ... 255] = -1,
    ['A'] = 0, ['a'] = 0, ['C'] = 1, ['c'] = 1, ['G'] = 2, ['g'] = 2, ['T'] = 3, ['t'] = 3,
    ['U'] = 4, ['N'] = 4, ['R'] = 4, ['Y'] = 4, ['S'] = 4, ['W'] = 4, ['K'] = 4, ['M'] = 4,
    ['B'] = 4, ['D'] = 4, ['H'] = 4, ['V'] = 4, ['u'] = 4, ['n'] = 4, ['r'] = 4, ['y'] = 4,
    ['s'] = 4, ['w'] = 4, ['k'] = 4, ['m'] = 4, ['b'] = 4, ['d'] = 4, ['h'] = 4, ['v'] = 4,
};

int or_char_to_code(char c) {
    return g_code[(unsigned char)c];
}

/* REF src/genome.cpp:39-46 append_base: code at bits (pos&31)*2 of word
 * pos>>5, N stored as code 0 plus bit pos&63 of mask word pos>>6. */
int or_pack_genome(const char* seq, uint64_t len, uint64_t* packed, uint64_t* nmask) {
    memset(packed, 0, ((len + 31) / 32) * sizeof(uint64_t));
    memset(nmask, 0, ((len + 63) / 64) * sizeof(uint64_t));
    for (uint64_t pos = 0; pos < len; ++pos) {
        int b = or_char_to_code(seq[pos]);
        if (b < 0) return -1;
        uint64_t code = b == 4 ? 0 : (uint64_t)b;
        packed[pos >> 5] |= code << ((pos & 31) * 2);
        if (b == 4) nmask[pos >> 6] |= (uint64_t)1 << (pos & 63);
    }
    return 0;
}

/* REF include/seedaln/genome.hpp:50-54 */
int or_genome_at(const or_genome* g, uint64_t pos) {
    uint64_t code = (g->packed[pos >> 5] >> ((pos & 31) * 2)) & 3;
    if ((g->nmask[pos >> 6] >> (pos & 63)) & 1) return 4;
    return (int)code;
}

static const char kBaseChars[5] = {'A', 'C', 'G', 'T', 'N'};

/* REF src/genome.cpp:114-123 substring: truncated at the genome end. */
static uint64_t genome_substring(const or_genome* g, uint64_t pos, uint64_t len, char* out) {
    uint64_t n = len < g->len - pos ? len : g->len - pos;
    for (uint64_t i = 0; i < n; ++i) out[i] = kBaseChars[or_genome_at(g, pos + i)];
    return n;
}

/* REF src/genome.cpp:182-200 reverse_complement; -1 on a non-ACGTN char. */
static int reverse_complement(const char* s, uint64_t n, char* out) {
    for (uint64_t i = 0; i < n; ++i) {
        char c;
        switch (s[n - 1 - i]) {
            case 'A': c = 'T'; break;
            case 'C': c = 'G'; break;
            case 'G': c = 'C'; break;
            case 'T': c = 'A'; break;
            case 'N': c = 'N'; break;
            default: return -1;
        }
        out[i] = c;
    }
    return 0;
}

/* ------------------------------------------------------------ seeds */

/* REF src/aligner.cpp:50-79 seed_offsets. */
int or_seed_offsets(uint64_t read_length, int s, int n, int* out) {
    int cnt = 0;
    if (s < 1 || n < 1 || read_length < (uint64_t)s) return 0;
    const int max_off = (int)read_length - s;
    char* seen = (char*)calloc((size_t)max_off + 1, 1);
#define EMIT_TIER(shift_)                                              \
    do {                                                               \
        for (int o = (shift_); o <= max_off && cnt < n; o += s) {      \
            if (!seen[o]) {                                            \
                seen[o] = 1;                                           \
                out[cnt++] = o;                                        \
            }                                                          \
        }                                                              \
    } while (0)
    EMIT_TIER(0);
    for (int level = 1; ((int64_t)1 << level) <= 4 * (int64_t)s && cnt < n; ++level) {
        for (int64_t odd = 1; odd < ((int64_t)1 << level) && cnt < n; odd += 2) {
            EMIT_TIER((int)((odd * s) >> level));
        }
    }
#undef EMIT_TIER
    free(seen);
    return cnt;
}

/* REF src/seed_index.cpp:51-60 pack_seed: first base in the high bits. */
int or_pack_seed(const char* seed, int s, uint64_t* out) {
    uint64_t key = 0;
    for (int i = 0; i < s; ++i) {
        int b = or_char_to_code(seed[i]);
        if (b < 0 || b == 4) return 0;
        key = (key << 2) | (uint64_t)b;
    }
    *out = key;
    return 1;
}

/* REF src/seed_index.cpp:62-70 packed_reverse_complement. */
uint64_t or_packed_rc(uint64_t key, int s) {
    uint64_t x = ~key;
    x = ((x & 0x3333333333333333ull) << 2) | ((x >> 2) & 0x3333333333333333ull);
    x = ((x & 0x0f0f0f0f0f0f0f0full) << 4) | ((x >> 4) & 0x0f0f0f0f0f0f0f0full);
    x = __builtin_bswap64(x);
    return x >> (64 - 2 * s);
}

/* ------------------------------------------------------------ index */

/* Stable LSD radix sort of (key, pos) by key over `bits` low bits; input in
 * position order, so equal keys keep ascending positions -- the same order
 * std::sort of (key, pos) pairs gives in REF seed_index.cpp:112. */
static int radix_sort_pairs(uint64_t* keys, uint32_t* pos, uint64_t n, int bits) {
    if (n < 2) return 0;
    uint64_t* k2 = (uint64_t*)malloc(n * sizeof(uint64_t));
    uint32_t* p2 = (uint32_t*)malloc(n * sizeof(uint32_t));
    size_t* hist = (size_t*)malloc((1u << 16) * sizeof(size_t));
    if (!k2 || !p2 || !hist) {
        free(k2); free(p2); free(hist);
        return -1;
    }
    uint64_t *ka = keys, *kb = k2;
    uint32_t *pa = pos, *pb = p2;
    for (int shift = 0; shift < bits; shift += 16) {
        memset(hist, 0, (1u << 16) * sizeof(size_t));
        for (uint64_t i = 0; i < n; ++i) hist[(ka[i] >> shift) & 0xffff]++;
        size_t sum = 0;
        for (int d = 0; d < (1 << 16); ++d) {
            size_t c = hist[d];
            hist[d] = sum;
            sum += c;
        }
        for (uint64_t i = 0; i < n; ++i) {
            size_t at = hist[(ka[i] >> shift) & 0xffff]++;
            kb[at] = ka[i];
            pb[at] = pa[i];
        }
        uint64_t* tk = ka; ka = kb; kb = tk;
        uint32_t* tp = pa; pa = pb; pb = tp;
    }
    if (ka != keys) {
        memcpy(keys, ka, n * sizeof(uint64_t));
        memcpy(pos, pa, n * sizeof(uint32_t));
    }
    free(k2); free(p2); free(hist);
    return 0;
}

static int radix_sort_keys(uint64_t* keys, uint64_t n, int bits) {
    if (n < 2) return 0;
    uint64_t* k2 = (uint64_t*)malloc(n * sizeof(uint64_t));
    size_t* hist = (size_t*)malloc((1u << 16) * sizeof(size_t));
    if (!k2 || !hist) {
        free(k2); free(hist);
        return -1;
    }
    uint64_t *ka = keys, *kb = k2;
    for (int shift = 0; shift < bits; shift += 16) {
        memset(hist, 0, (1u << 16) * sizeof(size_t));
        for (uint64_t i = 0; i < n; ++i) hist[(ka[i] >> shift) & 0xffff]++;
        size_t sum = 0;
        for (int d = 0; d < (1 << 16); ++d) {
            size_t c = hist[d];
            hist[d] = sum;
            sum += c;
        }
        for (uint64_t i = 0; i < n; ++i) kb[hist[(ka[i] >> shift) & 0xffff]++] = ka[i];
        uint64_t* t = ka; ka = kb; kb = t;
    }
    if (ka != keys) memcpy(keys, ka, n * sizeof(uint64_t));
    free(k2); free(hist);
    return 0;
}

/* REF src/seed_index.cpp:80-126 SeedIndex::build. */
int or_index_build(const or_genome* g, int seed_size, or_index* idx) {
    memset(idx, 0, sizeof(*idx));
    if (seed_size < 1 || seed_size > 32) return SA_EINVAL;
    if (g->len < (uint64_t)seed_size) return SA_EINVAL;
    if (g->len > 0xffffffffull) return SA_EINVAL;
    idx->seed_size = seed_size;
    const uint64_t s = (uint64_t)seed_size;
    const uint64_t mask = s == 32 ? ~(uint64_t)0 : (((uint64_t)1 << (2 * s)) - 1);

    uint64_t cap = g->len - s + 1;
    uint64_t* keys = (uint64_t*)malloc(cap * sizeof(uint64_t));
    uint32_t* pos = (uint32_t*)malloc(cap * sizeof(uint32_t));
    if (!keys || !pos) {
        free(keys); free(pos);
        return SA_ERUNTIME;
    }
    uint64_t n = 0, key = 0;
    int64_t last_n = -1;
    for (uint64_t p = 0; p < g->len; ++p) { /* REF :96-110 rolling key */
        int b = or_genome_at(g, p);
        if (b == 4) {
            last_n = (int64_t)p;
            key = (key << 2) & mask;
            continue;
        }
        key = ((key << 2) | (uint64_t)b) & mask;
        if (p + 1 < s) continue;
        uint64_t start = p + 1 - s;
        if ((int64_t)start <= last_n) continue;
        keys[n] = key;
        pos[n] = (uint32_t)start;
        n++;
    }
    if (radix_sort_pairs(keys, pos, n, (int)(2 * s)) != 0) {
        free(keys); free(pos);
        return SA_ERUNTIME;
    }
    /* CSR, REF :114-124 */
    uint64_t nk = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (i == 0 || keys[i] != keys[i - 1]) nk++;
    idx->keys = (uint64_t*)malloc((nk ? nk : 1) * sizeof(uint64_t));
    idx->offsets = (uint64_t*)malloc((nk + 1) * sizeof(uint64_t));
    uint64_t j = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (i == 0 || keys[i] != keys[i - 1]) {
            idx->keys[j] = keys[i];
            idx->offsets[j] = i;
            j++;
        }
    }
    idx->offsets[nk] = n;
    free(keys);
    idx->positions = pos;
    idx->n_keys = nk;
    idx->n_positions = n;
    return 0;
}

/* ---- query-restricted build (test infrastructure for 3.1 Gbp configs) */

static inline uint64_t mix_key(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    return x ^ (x >> 33);
}

typedef struct {
    const or_genome* g;
    uint64_t s, mask, begin, end; /* windows [begin, end) */
    const uint64_t* set;          /* open addressing, ~0 = empty */
    uint64_t set_mask;
    const uint64_t* filter;       /* 1 bit per hash bucket */
    uint64_t filter_mask;
    uint64_t* keys;               /* matches, grown as needed */
    uint32_t* pos;
    uint64_t n, cap;
    int failed;
} scan_job;

static int set_contains(const uint64_t* set, uint64_t set_mask, uint64_t key) {
    for (uint64_t h = mix_key(key) & set_mask;; h = (h + 1) & set_mask) {
        if (set[h] == key) return 1;
        if (set[h] == ~(uint64_t)0) return 0;
    }
}

static int scan_push(scan_job* j, uint64_t key, uint64_t start) {
    if (j->n == j->cap) {
        uint64_t nc = j->cap ? 2 * j->cap : 1 << 16;
        uint64_t* nk = (uint64_t*)realloc(j->keys, nc * sizeof(uint64_t));
        if (nk) j->keys = nk;
        uint32_t* np = (uint32_t*)realloc(j->pos, nc * sizeof(uint32_t));
        if (np) j->pos = np;
        if (!nk || !np) {
            j->failed = 1;
            return -1;
        }
        j->cap = nc;
    }
    j->keys[j->n] = key;
    j->pos[j->n] = (uint32_t)start;
    j->n++;
    return 0;
}

/* REF seed_index.cpp:96-110 rolling key, over windows [begin, end) only.
 * Each window costs a random filter access (and, when the filter says
 * maybe, a random set access): both are software-prefetched a fixed number
 * of windows ahead, so a thread keeps ~kPf misses in flight instead of one.
 * Windows are emitted in position order either way. */
#define kPf 32
static void* scan_windows(void* arg) {
    scan_job* j = (scan_job*)arg;
    uint64_t key = 0;
    int64_t last_n = -1;
    const uint64_t from = j->begin;
    const uint64_t to = j->end + j->s - 1; /* last base of the last window */
    /* stage 1: windows whose filter line is in flight; stage 2: filter hits
     * whose set slot is in flight */
    uint64_t k1[kPf], s1[kPf], h1[kPf], k2[kPf], s2[kPf];
    unsigned n1 = 0, t1 = 0, n2 = 0, t2 = 0;
    for (uint64_t p = from;; ++p) {
        const int more = p < to && p < j->g->len;
        if (more) {
            int b = or_genome_at(j->g, p);
            if (b == 4) {
                last_n = (int64_t)p;
                key = (key << 2) & j->mask;
                continue;
            }
            key = ((key << 2) | (uint64_t)b) & j->mask;
            if (p + 1 < from + j->s) continue;
            const uint64_t start = p + 1 - j->s;
            if ((int64_t)start <= last_n) continue;
            const uint64_t h = mix_key(key);
            __builtin_prefetch(&j->filter[(h >> 6) & j->filter_mask]);
            const unsigned at = (t1 + n1) % kPf;
            k1[at] = key;
            s1[at] = start;
            h1[at] = h;
            ++n1;
        }
        /* drain stage 1 when full (or at the end) */
        while (n1 == kPf || (!more && n1)) {
            const uint64_t h = h1[t1];
            if ((j->filter[(h >> 6) & j->filter_mask] >> (h & 63)) & 1) {
                while (n2 == kPf) { /* drain the oldest stage-2 entry */
                    if (set_contains(j->set, j->set_mask, k2[t2]) && scan_push(j, k2[t2], s2[t2])) return NULL;
                    t2 = (t2 + 1) % kPf;
                    --n2;
                }
                __builtin_prefetch(&j->set[h & j->set_mask]);
                const unsigned at = (t2 + n2) % kPf;
                k2[at] = k1[t1];
                s2[at] = s1[t1];
                ++n2;
            }
            t1 = (t1 + 1) % kPf;
            --n1;
            if (more) break;
        }
        if (!more) break;
    }
    while (n2) {
        if (set_contains(j->set, j->set_mask, k2[t2]) && scan_push(j, k2[t2], s2[t2])) return NULL;
        t2 = (t2 + 1) % kPf;
        --n2;
    }
    return NULL;
}

int or_index_build_for_reads(const or_genome* g, int seed_size, int n_seeds, const char* bases,
                             const uint64_t* offsets, uint64_t n_reads, int threads, or_index* idx) {
    memset(idx, 0, sizeof(*idx));
    if (seed_size < 1 || seed_size > 32 || n_seeds < 1) return SA_EINVAL;
    if (g->len < (uint64_t)seed_size || g->len > 0xffffffffull) return SA_EINVAL;
    if (threads < 1) threads = 1;
    idx->seed_size = seed_size;
    const uint64_t s = (uint64_t)seed_size;

    /* every key align() can probe (REF aligner.cpp:256-265, seed_index.cpp:128-143) */
    uint64_t nq = 0, qcap = 1 << 12;
    uint64_t* q = (uint64_t*)malloc(qcap * sizeof(uint64_t));
    int* offs = (int*)malloc((size_t)n_seeds * sizeof(int));
    if (!q || !offs) {
        free(q); free(offs);
        return SA_ERUNTIME;
    }
    uint64_t last_len = ~(uint64_t)0;
    int k = 0;
    for (uint64_t r = 0; r < n_reads; ++r) {
        const uint64_t len = offsets[r + 1] - offsets[r];
        if (len != last_len) { /* same offsets for every read of one length */
            k = or_seed_offsets(len, seed_size, n_seeds, offs);
            last_len = len;
        }
        for (int i = 0; i < k; ++i) {
            uint64_t key;
            if (!or_pack_seed(bases + offsets[r] + offs[i], seed_size, &key)) continue;
            if (nq + 2 > qcap) {
                qcap *= 2;
                uint64_t* nq2 = (uint64_t*)realloc(q, qcap * sizeof(uint64_t));
                if (!nq2) {
                    free(q); free(offs);
                    return SA_ERUNTIME;
                }
                q = nq2;
            }
            q[nq++] = key;
            q[nq++] = or_packed_rc(key, seed_size);
        }
    }
    free(offs);
    if (radix_sort_keys(q, nq, (int)(2 * s)) != 0) {
        free(q);
        return SA_ERUNTIME;
    }
    uint64_t u = 0;
    for (uint64_t i = 0; i < nq; ++i)
        if (u == 0 || q[i] != q[u - 1]) q[u++] = q[i];
    idx->queries = q;
    idx->n_queries = u;

    uint64_t set_size = 64;
    while (set_size < 4 * u) set_size <<= 1;
    uint64_t filter_words = 1024;
    while (filter_words * 64 < 16 * u) filter_words <<= 1;
    uint64_t* set = (uint64_t*)malloc(set_size * sizeof(uint64_t));
    uint64_t* filter = (uint64_t*)calloc(filter_words, sizeof(uint64_t));
    scan_job* jobs = (scan_job*)calloc((size_t)threads, sizeof(scan_job));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    if (!set || !filter || !jobs || !th) {
        free(set); free(filter); free(jobs); free(th);
        or_index_free(idx);
        return SA_ERUNTIME;
    }
    memset(set, 0xff, set_size * sizeof(uint64_t));
    for (uint64_t i = 0; i < u; ++i) {
        const uint64_t h = mix_key(q[i]);
        filter[(h >> 6) & (filter_words - 1)] |= (uint64_t)1 << (h & 63);
        uint64_t at = h & (set_size - 1);
        while (set[at] != ~(uint64_t)0) at = (at + 1) & (set_size - 1);
        set[at] = q[i];
    }

    const uint64_t n_windows = g->len - s + 1;
    for (int t = 0; t < threads; ++t) {
        scan_job* j = &jobs[t];
        j->g = g;
        j->s = s;
        j->mask = s == 32 ? ~(uint64_t)0 : (((uint64_t)1 << (2 * s)) - 1);
        j->begin = n_windows * (uint64_t)t / (uint64_t)threads;
        j->end = n_windows * (uint64_t)(t + 1) / (uint64_t)threads;
        j->set = set;
        j->set_mask = set_size - 1;
        j->filter = filter;
        j->filter_mask = filter_words - 1;
        pthread_create(&th[t], NULL, scan_windows, j);
    }
    int failed = 0;
    uint64_t n = 0;
    for (int t = 0; t < threads; ++t) {
        pthread_join(th[t], NULL);
        failed |= jobs[t].failed;
        n += jobs[t].n;
    }
    free(set); free(filter); free(th);
    /* concatenated in chunk order = genome position order, then the same
     * stable sort and CSR as or_index_build (REF seed_index.cpp:112-124) */
    uint64_t* keys = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    uint32_t* pos = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    if (!failed && keys && pos) {
        uint64_t at = 0;
        for (int t = 0; t < threads; ++t) {
            if (jobs[t].n) {
                memcpy(keys + at, jobs[t].keys, jobs[t].n * sizeof(uint64_t));
                memcpy(pos + at, jobs[t].pos, jobs[t].n * sizeof(uint32_t));
            }
            at += jobs[t].n;
        }
    }
    for (int t = 0; t < threads; ++t) {
        free(jobs[t].keys);
        free(jobs[t].pos);
    }
    free(jobs);
    if (failed || !keys || !pos || radix_sort_pairs(keys, pos, n, (int)(2 * s)) != 0) {
        free(keys); free(pos);
        or_index_free(idx);
        return SA_ERUNTIME;
    }
    uint64_t nk = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (i == 0 || keys[i] != keys[i - 1]) nk++;
    idx->keys = (uint64_t*)malloc((nk ? nk : 1) * sizeof(uint64_t));
    idx->offsets = (uint64_t*)malloc((nk + 1) * sizeof(uint64_t));
    uint64_t j = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (i == 0 || keys[i] != keys[i - 1]) {
            idx->keys[j] = keys[i];
            idx->offsets[j] = i;
            j++;
        }
    }
    idx->offsets[nk] = n;
    free(keys);
    idx->positions = pos;
    idx->n_keys = nk;
    idx->n_positions = n;
    return 0;
}

void or_index_free(or_index* idx) {
    free(idx->queries);
    free(idx->keys);
    free(idx->offsets);
    free(idx->positions);
    memset(idx, 0, sizeof(*idx));
}

/* std::lower_bound probe, REF seed_index.cpp:131-138. */
static void probe(const or_index* idx, uint64_t key, const uint32_t** span, uint64_t* len) {
    if (idx->queries) { /* restricted index: the key must be one it was built for */
        uint64_t a = 0, b = idx->n_queries;
        while (a < b) {
            uint64_t mid = a + (b - a) / 2;
            if (idx->queries[mid] < key) a = mid + 1;
            else b = mid;
        }
        if (a == idx->n_queries || idx->queries[a] != key)
            __atomic_fetch_add(&((or_index*)idx)->misses, 1, __ATOMIC_RELAXED);
    }
    uint64_t lo = 0, hi = idx->n_keys;
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (idx->keys[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    if (lo == idx->n_keys || idx->keys[lo] != key) {
        *span = NULL;
        *len = 0;
        return;
    }
    *span = idx->positions + idx->offsets[lo];
    *len = idx->offsets[lo + 1] - idx->offsets[lo];
}

/* REF src/seed_index.cpp:128-143 SeedIndex::lookup. */
int or_lookup(const or_index* idx, const char* seed, const uint32_t** fwd, uint64_t* n_fwd,
              const uint32_t** rc, uint64_t* n_rc) {
    uint64_t key;
    *fwd = *rc = NULL;
    *n_fwd = *n_rc = 0;
    if (!or_pack_seed(seed, idx->seed_size, &key)) return 0;
    probe(idx, key, fwd, n_fwd);
    probe(idx, or_packed_rc(key, idx->seed_size), rc, n_rc);
    return 0;
}

/* ------------------------------------------------------------ LV */

/* REF src/edit_distance.cpp:11-13: N never matches, even N-N. */
static inline int bases_match(char a, char b) { return a == b && a != 'N' && b != 'N'; }

#define K_UNREACHABLE (INT64_MIN / 2)

/* REF src/edit_distance.cpp:19-75 bounded_distance. */
int or_bounded_distance(const char* read, int64_t m, const char* win, int64_t w, int d_limit,
                        uint64_t* cells) {
    if (d_limit < 0) return -2;
    uint64_t touched = 0;
    const int64_t off = d_limit + 1;
    const int64_t sz = 2 * (int64_t)d_limit + 3;
    int64_t* best = (int64_t*)malloc(sz * sizeof(int64_t));
    int64_t* next = (int64_t*)malloc(sz * sizeof(int64_t));
    for (int64_t i = 0; i < sz; ++i) best[i] = next[i] = K_UNREACHABLE;

    int result = -1;
    for (int e = 0; e <= d_limit && result < 0; ++e) {
        for (int64_t k = -e; k <= e; ++k) {
            if (k > w) continue;
            int64_t cand;
            if (e == 0) {
                cand = 0;
            } else {
                cand = best[k + off] + 1;
                int64_t c2 = best[k + 1 + off] + 1;
                if (c2 > cand) cand = c2;
                int64_t c3 = best[k - 1 + off];
                if (c3 > cand) cand = c3;
            }
            int64_t lowest = -k > 0 ? -k : 0;
            if (cand < lowest) {
                next[k + off] = K_UNREACHABLE;
                continue;
            }
            int64_t cap = m < w - k ? m : w - k;
            if (cand > cap) cand = cap;
            while (cand < cap && bases_match(read[cand], win[cand + k])) { /* slide */
                ++cand;
                ++touched;
            }
            ++touched;
            next[k + off] = cand;
            if (cand == m) {
                result = e;
                break;
            }
        }
        int64_t* t = best; best = next; next = t;
    }
    free(best);
    free(next);
    if (cells) *cells += touched;
    return result;
}

/* REF src/edit_distance.cpp:77-95 full_dp_distance. */
int or_full_dp_distance(const char* read, int64_t m, const char* win, int64_t w) {
    int* row = (int*)calloc((size_t)w + 1, sizeof(int));
    int* prev = (int*)calloc((size_t)w + 1, sizeof(int));
    for (int64_t j = 0; j <= w; ++j) prev[j] = (int)j;
    for (int64_t i = 1; i <= m; ++i) {
        row[0] = (int)i;
        for (int64_t j = 1; j <= w; ++j) {
            int sub = prev[j - 1] + (bases_match(read[i - 1], win[j - 1]) ? 0 : 1);
            int v = sub;
            if (prev[j] + 1 < v) v = prev[j] + 1;
            if (row[j - 1] + 1 < v) v = row[j - 1] + 1;
            row[j] = v;
        }
        int* t = row; row = prev; prev = t;
    }
    int best = prev[0];
    for (int64_t j = 1; j <= w; ++j)
        if (prev[j] < best) best = prev[j];
    free(row);
    free(prev);
    return best;
}

/* ------------------------------------------------------------ aligner */

/* BestTracker, REF aligner.hpp:82-101 / aligner.cpp:87-114. */
typedef struct tracker {
    int merge_radius;
    int d_best, d_second;
    uint64_t best_position;
    int best_direction;
} tracker;

static void tracker_observe(tracker* t, int distance, uint64_t position, int direction) {
    if (t->d_best < K_INF_DISTANCE && direction == t->best_direction) {
        uint64_t delta = position > t->best_position ? position - t->best_position
                                                     : t->best_position - position;
        if (delta <= (uint64_t)t->merge_radius) {
            if (distance < t->d_best) {
                t->d_best = distance;
                t->best_position = position;
            }
            return;
        }
    }
    if (distance < t->d_best) {
        t->d_second = t->d_best;
        t->d_best = distance;
        t->best_position = position;
        t->best_direction = direction;
    } else if (distance < t->d_second) {
        t->d_second = distance;
    }
}

static int tracker_gap(const tracker* t) {
    if (t->d_second >= K_INF_DISTANCE) return K_GAP_CAP;
    int g = t->d_second - t->d_best;
    return g < K_GAP_CAP ? g : K_GAP_CAP;
}

/* Candidate, REF aligner.hpp:128-134 */
typedef struct candidate {
    uint64_t bucket;
    int dir;
    uint32_t seeds_hitting;
    uint64_t anchor_mask;
    int scored;
} candidate;

typedef struct scratch {
    candidate* cands;
    size_t n_cands, cap_cands;
    /* bucket_map_ (unordered_map<uint64,uint32>) restated as open addressing */
    uint64_t* hkeys;
    uint32_t* hvals;
    size_t hcap; /* power of two */
    char* rc;
    char* window;
    size_t rc_cap, win_cap;
    int* offsets;
    size_t off_cap;
    /* per-read state, REF aligner.hpp:150-157 */
    uint64_t calls_this_read;
    int first_scored_done, first_locus_valid, first_locus_dir;
    uint64_t first_locus_pos;
} scratch;

static void scratch_free(scratch* sc) {
    free(sc->cands);
    free(sc->hkeys);
    free(sc->hvals);
    free(sc->rc);
    free(sc->window);
    free(sc->offsets);
}

static void map_clear(scratch* sc) {
    if (!sc->hkeys) {
        sc->hcap = 64;
        sc->hkeys = (uint64_t*)malloc(sc->hcap * sizeof(uint64_t));
        sc->hvals = (uint32_t*)malloc(sc->hcap * sizeof(uint32_t));
    }
    memset(sc->hkeys, 0xff, sc->hcap * sizeof(uint64_t));
    sc->n_cands = 0;
}

static inline size_t hash_slot(uint64_t key, size_t hcap) {
    return (size_t)((key * 0x9E3779B97F4A7C15ull) >> 17) & (hcap - 1);
}

static void map_grow(scratch* sc) {
    size_t ncap = sc->hcap * 2;
    uint64_t* nk = (uint64_t*)malloc(ncap * sizeof(uint64_t));
    uint32_t* nv = (uint32_t*)malloc(ncap * sizeof(uint32_t));
    memset(nk, 0xff, ncap * sizeof(uint64_t));
    for (size_t i = 0; i < sc->hcap; ++i) {
        if (sc->hkeys[i] == ~(uint64_t)0) continue;
        size_t h = hash_slot(sc->hkeys[i], ncap);
        while (nk[h] != ~(uint64_t)0) h = (h + 1) & (ncap - 1);
        nk[h] = sc->hkeys[i];
        nv[h] = sc->hvals[i];
    }
    free(sc->hkeys);
    free(sc->hvals);
    sc->hkeys = nk;
    sc->hvals = nv;
    sc->hcap = ncap;
}

/* REF aligner.cpp:124-134 add_hit */
static void add_hit(scratch* sc, uint64_t anchor, int dir, uint64_t bs) {
    uint64_t bucket = anchor / bs;
    uint64_t key = bucket * 2 + (uint64_t)dir;
    if ((sc->n_cands + 1) * 2 > sc->hcap) map_grow(sc);
    size_t h = hash_slot(key, sc->hcap);
    while (sc->hkeys[h] != ~(uint64_t)0 && sc->hkeys[h] != key) h = (h + 1) & (sc->hcap - 1);
    if (sc->hkeys[h] == ~(uint64_t)0) { /* try_emplace inserted */
        if (sc->n_cands == sc->cap_cands) {
            sc->cap_cands = sc->cap_cands ? sc->cap_cands * 2 : 64;
            sc->cands = (candidate*)realloc(sc->cands, sc->cap_cands * sizeof(candidate));
        }
        sc->hkeys[h] = key;
        sc->hvals[h] = (uint32_t)sc->n_cands;
        candidate c = {bucket, dir, 0, 0, 0};
        sc->cands[sc->n_cands++] = c;
    }
    candidate* cand = &sc->cands[sc->hvals[h]];
    cand->seeds_hitting++;
    cand->anchor_mask |= (uint64_t)1 << (anchor - bucket * bs);
}

/* REF aligner.cpp:136-139 has_unscored */
static int has_unscored(const scratch* sc) {
    for (size_t i = 0; i < sc->n_cands; ++i)
        if (!sc->cands[i].scored) return 1;
    return 0;
}

typedef struct read_ctx {
    const or_genome* g;
    const sa_params* p;
    const char* bases;
    const char* rc;
    uint64_t len;
    int d_max;
    tracker* tr;
    sa_stats* st;
} read_ctx;

/* REF aligner.cpp:169-221 score_candidate */
static void score_candidate(scratch* sc, candidate* cand, read_ctx* r) {
    cand->scored = 1;
    const int c = r->p->confidence_threshold;
    const int d_max = r->d_max;
    int d_limit;
    if (r->tr->d_best > d_max) d_limit = d_max + c - 1;
    else if (r->tr->d_second >= r->tr->d_best + c) d_limit = r->tr->d_best + c - 1;
    else d_limit = r->tr->d_best - 1;
    if (r->p->force_max_dlimit) d_limit = d_max + c - 1;
    if (d_limit < 0) return;

    const char* oriented = cand->dir == 0 ? r->bases : r->rc;
    const uint64_t bs = (uint64_t)r->p->bucket_size;
    const uint64_t base_pos = cand->bucket * bs;
    size_t need = r->len + (size_t)d_limit + 1;
    if (need > sc->win_cap) {
        sc->win_cap = need;
        sc->window = (char*)realloc(sc->window, need);
    }
    int best_d = K_INF_DISTANCE;
    uint64_t best_anchor = 0;
    for (uint64_t mask = cand->anchor_mask; mask != 0; mask &= mask - 1) {
        uint64_t anchor = base_pos + (uint64_t)__builtin_ctzll(mask);
        if (anchor >= r->g->len) continue;
        uint64_t w = genome_substring(r->g, anchor, r->len + (uint64_t)d_limit, sc->window);
        int out = or_bounded_distance(oriented, (int64_t)r->len, sc->window, (int64_t)w, d_limit,
                                      &r->st->dp_cells);
        r->st->distance_calls++;
        sc->calls_this_read++;
        r->st->window_bases += w;
        if (sc->calls_this_read > 1) {
            r->st->distance_calls_after_first++;
            if (out < 0) r->st->early_out_after_first++;
        }
        if (out >= 0 && out < best_d) {
            best_d = out;
            best_anchor = anchor;
        }
    }
    if (!sc->first_scored_done) {
        sc->first_scored_done = 1;
        if (best_d < K_INF_DISTANCE) {
            sc->first_locus_valid = 1;
            sc->first_locus_pos = best_anchor;
            sc->first_locus_dir = cand->dir;
        }
    }
    if (best_d < K_INF_DISTANCE) tracker_observe(r->tr, best_d, best_anchor, cand->dir);
}

/* REF aligner.cpp:141-167 score_best_candidate */
static void score_best_candidate(scratch* sc, read_ctx* r) {
    candidate* best = NULL;
    uint64_t best_amin = 0;
    const uint64_t bs = (uint64_t)r->p->bucket_size;
    for (size_t i = 0; i < sc->n_cands; ++i) {
        candidate* cand = &sc->cands[i];
        if (cand->scored) continue;
        uint64_t amin = cand->bucket * bs + (uint64_t)__builtin_ctzll(cand->anchor_mask);
        int better;
        if (!best) better = 1;
        else if (cand->seeds_hitting != best->seeds_hitting)
            better = cand->seeds_hitting > best->seeds_hitting;
        else if (amin != best_amin)
            better = amin < best_amin;
        else
            better = cand->dir < best->dir;
        if (better) {
            best = cand;
            best_amin = amin;
        }
    }
    if (best) score_candidate(sc, best, r);
}

static int validate(const sa_params* p) {
    if (p->seed_size < 1 || p->seed_size > 32) return SA_EINVAL;
    if (p->seeds_to_try < 1) return SA_EINVAL;
    if (p->max_distance < -1) return SA_EINVAL;
    if (p->confidence_threshold < 1) return SA_EINVAL;
    if (p->max_hits < 1) return SA_EINVAL;
    if (p->bucket_size < 1 || p->bucket_size > 64) return SA_EINVAL;
    return 0;
}

/* REF aligner.cpp:223-364 Aligner::align */
static int align_one(scratch* sc, const or_index* idx, const or_genome* g, const sa_params* p,
                     const char* bases, uint64_t len, sa_result* result, sa_stats* st) {
    st->reads++;
    st->read_bases += len;
    const int s = p->seed_size;
    memset(result, 0, sizeof(*result));
    result->kind = SA_NOT_FOUND;
    result->distance = -1;
    if (len < (uint64_t)s) {
        st->reads_too_short++;
        st->not_found++;
        return 0;
    }
    const int d_max = p->max_distance >= 0 ? p->max_distance : (int)((12 * len + 99) / 100);
    const int c = p->confidence_threshold;
    if ((size_t)p->seeds_to_try > sc->off_cap) {
        sc->off_cap = (size_t)p->seeds_to_try;
        sc->offsets = (int*)realloc(sc->offsets, sc->off_cap * sizeof(int));
    }
    const int n_off = or_seed_offsets(len, s, p->seeds_to_try, sc->offsets);
    const int tier0_count = (int)(len / (uint64_t)s);
    if (len + 1 > sc->rc_cap) {
        sc->rc_cap = len + 1;
        sc->rc = (char*)realloc(sc->rc, sc->rc_cap);
    }
    if (reverse_complement(bases, len, sc->rc) != 0) return SA_EINVAL;

    map_clear(sc);
    sc->calls_this_read = 0;
    sc->first_scored_done = 0;
    sc->first_locus_valid = 0;
    tracker tr = {p->bucket_size, K_INF_DISTANCE, K_INF_DISTANCE, 0, 0};
    read_ctx r = {g, p, bases, sc->rc, len, d_max, &tr, st};

    int tested_non_overlapping = 0;
    int any_lookup = 0, any_popular = 0, early_multi = 0;
    const uint64_t bs = (uint64_t)p->bucket_size;

    for (int i = 0; i < n_off; ++i) {
        const int off = sc->offsets[i];
        const char* seed = bases + off;
        if (memchr(seed, 'N', (size_t)s) != NULL) {
            st->seeds_skipped_n++;
            continue;
        }
        const uint32_t *fwd, *rcl;
        uint64_t nf, nr;
        or_lookup(idx, seed, &fwd, &nf, &rcl, &nr);
        st->seed_lookups++;
        if (nf + nr > (uint64_t)p->max_hits) {
            any_popular = 1;
            st->seeds_skipped_popular++;
            continue;
        }
        any_lookup = 1;
        st->hits_consumed += nf + nr;
        if (i < tier0_count) ++tested_non_overlapping;
        for (uint64_t j = 0; j < nf; ++j) {
            int64_t anchor = (int64_t)fwd[j] - off;
            add_hit(sc, anchor < 0 ? 0 : (uint64_t)anchor, 0, bs);
        }
        const int rc_shift = (int)len - s - off;
        for (uint64_t j = 0; j < nr; ++j) {
            int64_t anchor = (int64_t)rcl[j] - rc_shift;
            add_hit(sc, anchor < 0 ? 0 : (uint64_t)anchor, 1, bs);
        }
        score_best_candidate(sc, &r);
        if (tr.d_best < c && tr.d_second < tr.d_best + c) {
            st->multi_early_exits++;
            early_multi = 1;
            break;
        }
        if (tested_non_overlapping >= tr.d_best + c) {
            st->pruning_exits++;
            while (has_unscored(sc)) {
                score_best_candidate(sc, &r);
                if (tr.d_best < c && tr.d_second < tr.d_best + c) {
                    st->multi_early_exits++;
                    early_multi = 1;
                    break;
                }
            }
            break;
        }
    }

    int kind;
    if (early_multi) {
        kind = SA_MULTIPLE_HITS;
    } else {
        /* classify_confidence, REF aligner.cpp:81-85 */
        if (tr.d_best <= d_max && tr.d_second >= tr.d_best + c) kind = SA_SINGLE_HIT;
        else if (tr.d_best <= d_max) kind = SA_MULTIPLE_HITS;
        else kind = SA_NOT_FOUND;
        if (kind == SA_NOT_FOUND && any_popular && !any_lookup) {
            st->reads_all_seeds_popular++;
            kind = SA_MULTIPLE_HITS;
        }
    }
    result->kind = (uint8_t)kind;
    if (kind == SA_SINGLE_HIT) {
        result->has_position = 1;
        result->position = tr.best_position;
        result->direction = (uint8_t)tr.best_direction;
        result->distance = tr.d_best;
        result->gap = tracker_gap(&tr);
        st->single_hits++;
        if (sc->first_locus_valid && sc->first_locus_dir == tr.best_direction) {
            uint64_t delta = sc->first_locus_pos > tr.best_position
                                 ? sc->first_locus_pos - tr.best_position
                                 : tr.best_position - sc->first_locus_pos;
            if (delta <= bs) st->first_scored_was_best++;
        }
    } else if (kind == SA_MULTIPLE_HITS) {
        if (tr.d_best < K_INF_DISTANCE && tr.d_best <= d_max) {
            result->has_position = 1;
            result->position = tr.best_position;
            result->direction = (uint8_t)tr.best_direction;
            result->distance = tr.d_best;
            result->gap = tracker_gap(&tr);
        }
        st->multiple_hits++;
    } else {
        st->not_found++;
    }
    return 0;
}

int or_align(const or_index* idx, const or_genome* g, const sa_params* p, const char* bases,
             uint64_t len, sa_result* res, sa_stats* stats) {
    if (validate(p) != 0 || idx->seed_size != p->seed_size) return SA_EINVAL;
    scratch sc;
    memset(&sc, 0, sizeof(sc));
    sa_stats local;
    memset(&local, 0, sizeof(local));
    int rcode = align_one(&sc, idx, g, p, bases, len, res, &local);
    scratch_free(&sc);
    if (stats) {
        uint64_t* d = (uint64_t*)stats;
        const uint64_t* s = (const uint64_t*)&local;
        for (size_t i = 0; i < sizeof(sa_stats) / 8; ++i) d[i] += s[i];
    }
    return rcode;
}

typedef struct batch_job {
    const or_index* idx;
    const or_genome* g;
    const sa_params* p;
    const char* bases;
    const uint64_t* offsets;
    uint64_t n;
    sa_result* res;
    atomic_uint_fast64_t cursor;
    atomic_int failed;
    pthread_mutex_t mu;
    sa_stats total;
} batch_job;

static void* batch_worker(void* arg) {
    batch_job* job = (batch_job*)arg;
    scratch sc;
    memset(&sc, 0, sizeof(sc));
    sa_stats local;
    memset(&local, 0, sizeof(local));
    const uint64_t grain = 64;
    for (;;) {
        uint64_t begin = atomic_fetch_add(&job->cursor, grain);
        if (begin >= job->n || atomic_load(&job->failed)) break;
        uint64_t end = begin + grain < job->n ? begin + grain : job->n;
        for (uint64_t i = begin; i < end; ++i) {
            uint64_t o = job->offsets[i];
            if (align_one(&sc, job->idx, job->g, job->p, job->bases + o, job->offsets[i + 1] - o,
                          &job->res[i], &local) != 0) {
                atomic_store(&job->failed, 1);
                break;
            }
        }
    }
    scratch_free(&sc);
    pthread_mutex_lock(&job->mu);
    uint64_t* d = (uint64_t*)&job->total;
    const uint64_t* s = (const uint64_t*)&local;
    for (size_t i = 0; i < sizeof(sa_stats) / 8; ++i) d[i] += s[i];
    pthread_mutex_unlock(&job->mu);
    return NULL;
}

int or_align_batch(const or_index* idx, const or_genome* g, const sa_params* p,
                   const char* bases, const uint64_t* offsets, uint64_t n, sa_result* res,
                   sa_stats* stats, int threads) {
    if (validate(p) != 0 || idx->seed_size != p->seed_size) return SA_EINVAL;
    if (threads < 1) threads = 1;
    batch_job job;
    memset(&job, 0, sizeof(job));
    job.idx = idx;
    job.g = g;
    job.p = p;
    job.bases = bases;
    job.offsets = offsets;
    job.n = n;
    job.res = res;
    atomic_init(&job.cursor, 0);
    atomic_init(&job.failed, 0);
    pthread_mutex_init(&job.mu, NULL);
    if (threads == 1) {
        batch_worker(&job);
    } else {
        pthread_t* th = (pthread_t*)malloc((size_t)threads * sizeof(pthread_t));
        for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, batch_worker, &job);
        for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
        free(th);
    }
    pthread_mutex_destroy(&job.mu);
    if (stats) {
        uint64_t* d = (uint64_t*)stats;
        const uint64_t* s = (const uint64_t*)&job.total;
        for (size_t i = 0; i < sizeof(sa_stats) / 8; ++i) d[i] += s[i];
    }
    return atomic_load(&job.failed) ? SA_EINVAL : 0;
}
