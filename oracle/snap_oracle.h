/*
 * snap_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference's aligner hot path, used as the
 * parity checker for the CUDA path.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * (paper_1111_5572_b200) never links or calls it.
 *
 * Parity is pinned: tests/test_oracle.py checks this restatement against the
 * reference's own known-answer vectors (tests/golden/) and against the
 * reference library itself compiled from /root/reference (oracle/_ref).
 *
 * Types (sa_params / sa_result / sa_stats) are shared with the product header
 * so results compare field by field.
 */
#ifndef SNAP_ORACLE_H
#define SNAP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/snap_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Genome view in PackedGenome layout (REF include/seedaln/genome.hpp:50-54,82-83). */
typedef struct or_genome {
    uint64_t len;
    const uint64_t* packed; /* 32 bases / word, LSB-first */
    const uint64_t* nmask;  /* 64 positions / word        */
} or_genome;

/* CSR seed index (REF include/seedaln/seed_index.hpp:66-71): sorted distinct
 * keys, offsets (n_keys + 1), positions ascending per key.  Positions are
 * stored as uint32 (genomes < 2^32) -- values identical to the reference. */
typedef struct or_index {
    int seed_size;
    uint64_t n_keys;
    uint64_t n_positions;
    uint64_t* keys;
    uint64_t* offsets;
    uint32_t* positions;
    /* query-restricted index (or_index_build_for_reads): only the keys in
     * `queries` (sorted) are indexed; probing any other key counts a miss,
     * so a test can prove it never asked the restricted index an unknown key */
    uint64_t n_queries;
    uint64_t* queries;
    uint64_t misses;
} or_index;

int or_char_to_code(char c); /* 0..3 for ACGT (any case), 4 for IUPAC N-class, -1 illegal */

/* ASCII -> PackedGenome words (REF src/genome.cpp:39-46 append_base). */
int or_pack_genome(const char* seq, uint64_t len, uint64_t* packed, uint64_t* nmask);

int or_genome_at(const or_genome* g, uint64_t pos); /* REF genome.hpp:50-54; 4 = N */

int or_seed_offsets(uint64_t read_length, int s, int n, int* out); /* returns count */
int or_pack_seed(const char* seed, int s, uint64_t* out);          /* 1 ok, 0 has N/illegal */
uint64_t or_packed_rc(uint64_t key, int s);

int or_index_build(const or_genome* g, int seed_size, or_index* out); /* 0 ok */
void or_index_free(or_index* idx);
/* The same CSR restricted to every key a batch of reads can probe: the
 * packed key and packed RC of each N-free seed at seed_offsets(len, s,
 * n_seeds) of each read.  One threaded scan of the genome's windows collects
 * their positions, so 3.1 Gbp genomes index in seconds and little memory;
 * for those keys, lookup() answers exactly what or_index_build's would. */
int or_index_build_for_reads(const or_genome* g, int seed_size, int n_seeds, const char* bases,
                             const uint64_t* offsets, uint64_t n_reads, int threads, or_index* out);
/* REF seed_index.cpp:128-143: forward span and rc span into idx->positions. */
int or_lookup(const or_index* idx, const char* seed, const uint32_t** fwd, uint64_t* n_fwd,
              const uint32_t** rc, uint64_t* n_rc);

/* REF src/edit_distance.cpp:19-75.  Returns distance or -1 (nullopt);
 * -2 when d_limit < 0 (the reference throws). */
int or_bounded_distance(const char* read, int64_t m, const char* win, int64_t w, int d_limit,
                        uint64_t* cells);
int or_full_dp_distance(const char* read, int64_t m, const char* win, int64_t w);

/* Aligner::align, REF src/aligner.cpp:223-364.  Returns 0, or SA_EINVAL when
 * the read holds a character outside {A,C,G,T,N} (reference throws). */
int or_align(const or_index* idx, const or_genome* g, const sa_params* p, const char* bases,
             uint64_t len, sa_result* res, sa_stats* stats);

/* align_corpus pattern (REF tests/acceptance/acceptance_main.cpp:52-67,106-124):
 * `threads` workers, atomic cursor, grain 64. */
int or_align_batch(const or_index* idx, const or_genome* g, const sa_params* p,
                   const char* bases, const uint64_t* offsets, uint64_t n, sa_result* res,
                   sa_stats* stats, int threads);

#ifdef __cplusplus
}
#endif
#endif
