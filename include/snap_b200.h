/*
 * snap_b200.h -- C-ABI drop-in boundary for the SNAP aligner core on B200.
 *
 * The reference (`seedaln`, /root/reference/proj) exposes the hot path only as
 * a C++ library API.  Every entry point below replaces one reference call
 * site; the reference interface it stands in for is cited beside it
 * (REF = /root/reference/proj).  Plain pointers and sizes only: no C++, no
 * torch types.  Every function returns an int status:
 *
 *   SA_OK       0  success
 *   SA_EINVAL   1  invalid argument   (reference: std::invalid_argument)
 *   SA_ERUNTIME 2  CUDA / runtime      (reference: IoError / runtime_error)
 *   SA_EFORMAT  3  format mismatch     (reference: FormatError)
 *   SA_EPARSE   4  malformed text input (reference: ParseError, FASTA/FASTQ)
 *   SA_EIO      5  file cannot be opened/written (reference: IoError)
 *
 * and leaves a message retrievable with sa_last_error().  The C++ adapter in
 * snap_b200.hpp rethrows these as the reference's exception types.
 *
 * Ownership: the caller owns every host buffer it passes in; the library owns
 * all device memory and pinned staging it allocates.  A context may be used
 * from one thread at a time (calls on one context are serialised internally).
 */
#ifndef SNAP_B200_H
#define SNAP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SA_OK = 0, SA_EINVAL = 1, SA_ERUNTIME = 2, SA_EFORMAT = 3, SA_EPARSE = 4, SA_EIO = 5 };

/* ResultKind, REF include/seedaln/aligner.hpp:32 */
enum { SA_SINGLE_HIT = 0, SA_MULTIPLE_HITS = 1, SA_NOT_FOUND = 2 };
/* Direction, REF include/seedaln/seed_index.hpp:14 */
enum { SA_FORWARD = 0, SA_REVERSE_COMPLEMENT = 1 };

/* AlignerParams, REF include/seedaln/aligner.hpp:19-30 (same defaults via
 * sa_default_params; same validation rules, REF src/aligner.cpp:11-24). */
typedef struct sa_params {
    int32_t seed_size;            /* s: seed length in bases, [1, 32]        */
    int32_t seeds_to_try;         /* n: seeds drawn per read, >= 1           */
    int32_t max_distance;         /* d_max, -1 = ceil(0.12 * read length)    */
    int32_t confidence_threshold; /* c, >= 1                                 */
    int32_t max_hits;             /* h_max, >= 1                             */
    int32_t bucket_size;          /* [1, 64]                                 */
    int32_t force_max_dlimit;     /* bool: disable d_limit shrinking         */
} sa_params;

/* AlignmentResult, REF include/seedaln/aligner.hpp:36-44.  24 bytes. */
typedef struct sa_result {
    uint64_t position;     /* forward-strand start of the alignment          */
    int32_t distance;      /* edit distance of the best hit, -1 if none      */
    int32_t gap;           /* d_second - d_best capped at 1000 (kGapCap)     */
    uint8_t kind;          /* SA_SINGLE_HIT / SA_MULTIPLE_HITS / SA_NOT_FOUND */
    uint8_t has_position;  /* bool                                           */
    uint8_t direction;     /* SA_FORWARD / SA_REVERSE_COMPLEMENT             */
    uint8_t reserved[5];
} sa_result;

/* AlignStats, REF include/seedaln/aligner.hpp:47-66 (first 16 fields, same
 * order and meaning; dp_cells counts this implementation's LV cells), plus
 * path counters used for the algorithmic-byte roofline. */
typedef struct sa_stats {
    uint64_t reads;
    uint64_t reads_too_short;
    uint64_t seed_lookups;
    uint64_t seeds_skipped_n;
    uint64_t seeds_skipped_popular;
    uint64_t reads_all_seeds_popular;
    uint64_t distance_calls;
    uint64_t distance_calls_after_first;
    uint64_t early_out_after_first;
    uint64_t dp_cells;
    uint64_t multi_early_exits;
    uint64_t pruning_exits;
    uint64_t first_scored_was_best;
    uint64_t single_hits;
    uint64_t multiple_hits;
    uint64_t not_found;
    /* extensions (not in the reference's AlignStats) */
    uint64_t hits_consumed;  /* sum of hit counts of non-popular looked-up seeds */
    uint64_t window_bases;   /* sum over LV calls of the genome window length    */
    uint64_t read_bases;     /* sum of read lengths                              */
    uint64_t overflow_reads; /* reads re-run on the global candidate-table path  */
} sa_stats;

typedef struct sa_context sa_context;

/* Defaults of AlignerParams (REF aligner.hpp:20-26). */
void sa_default_params(sa_params* out);

/* AlignerParams::validate (REF src/aligner.cpp:11-24).  SA_EINVAL on failure. */
int sa_validate_params(const sa_params* p);

/* seed_offsets (REF src/aligner.cpp:50-79).  Writes up to n offsets into out
 * (capacity >= n) and stores the count in *count. Host-side, pure. */
int sa_seed_offsets(uint64_t read_length, int32_t s, int32_t n, int32_t* out,
                    int32_t* count);

/* Context = genome resident in HBM + GPU seed index, one replica per device.
 * Replaces SeedIndex::build(const PackedGenome&, int)   (REF src/seed_index.cpp:80-126)
 * and the Aligner constructor's index/genome binding     (REF src/aligner.cpp:116-122).
 * packed_words / nmask_words are exactly PackedGenome::packed_words() and
 * n_mask_words() (REF include/seedaln/genome.hpp:73-74,82-83): 32 bases per
 * word LSB-first (A=0 C=1 G=2 T=3), and one N bit per position.
 * devices: CUDA ordinals (NULL/0 = device 0 only).
 * Errors: SA_EINVAL when seed_size is outside [1,32], the genome is shorter
 * than seed_size (REF seed_index.cpp:81-84) or longer than 2^32-1 bases. */
int sa_create(const uint64_t* packed_words, uint64_t n_packed,
              const uint64_t* nmask_words, uint64_t n_nmask,
              uint64_t genome_length, int32_t seed_size,
              const int32_t* devices, int32_t n_devices, sa_context** out);

void sa_destroy(sa_context* ctx);

/* Message of the last failing call on ctx (ctx == NULL: last failing call of
 * this thread that had no context).  Never NULL. */
const char* sa_last_error(const sa_context* ctx);

/* Aligner::align over a batch (REF src/aligner.cpp:223-364, called per read
 * by the run_align worker REF src/driver.cpp:113).  Reads are ASCII over
 * {A,C,G,T,N}: read i is bases[offsets[i] .. offsets[i+1]).  results[i] is
 * the AlignmentResult of read i (input order).  stats (nullable) receives the
 * AlignStats summed over the batch (REF aligner.cpp:31-48 merge semantics).
 * Blocking.  Host buffers may be pageable or pinned (sa_host_alloc): pinned
 * reads are copied in chunk by chunk behind the kernels; pageable reads are
 * packed (2+1 bits per base) by the library's host threads into its own
 * pinned buffers first.  Either way copies overlap the kernels.
 * Errors: SA_EINVAL on invalid params, a seed-size mismatch with the index
 * (REF aligner.cpp:119-121), or a read of length >= s holding a character
 * outside {A,C,G,T,N} (REF genome.cpp:182-200 throws from align()). */
int sa_align_batch(sa_context* ctx, const sa_params* params, const char* bases,
                   const uint64_t* offsets, uint64_t n_reads, sa_result* results,
                   sa_stats* stats);

/* Same as sa_align_batch with every buffer already in device memory of the
 * context's first device (no host copies); stream is a cudaStream_t (0 =
 * legacy default).  max_read_length bounds every read's length (it sizes the
 * per-warp shared-memory layout).  Asynchronous: returns after enqueueing.
 * d_stats (device, nullable) is accumulated into, not overwritten.  Errors
 * found by the kernels (invalid characters) are reported by the next sa_sync().
 * Calls on one context share its device scratch: a call enqueued on a stream
 * other than the previous call's waits (on the device) for that call's work,
 * so concurrent calls are correct but do not overlap. */
int sa_align_device(sa_context* ctx, const sa_params* params, const char* d_bases,
                    const uint64_t* d_offsets, uint64_t n_reads, uint64_t max_read_length,
                    sa_result* d_results, sa_stats* d_stats, void* stream);

/* Waits for sa_align_device work on stream and reports deferred errors. */
int sa_sync(sa_context* ctx, void* stream);

/* SeedIndex::lookup over a batch (REF src/seed_index.cpp:128-143).  seeds holds
 * n_seeds ASCII seeds of exactly seed_size characters, back to back.
 * counts[i] = LookupResult::count() (forward + rc; a palindromic seed counts
 * twice, REF tests/test_seed_index.cpp:67-85).  If fwd_out/rc_out are non-NULL
 * the positions are written there: seed i's forward list at
 * fwd_out[i*cap ..] (ascending, at most cap entries) with its length in
 * n_fwd[i], likewise rc_out / n_rc.  Seeds with N or of unknown key -> 0. */
int sa_lookup_batch(sa_context* ctx, const char* seeds, uint64_t n_seeds,
                    uint32_t* counts, uint64_t* fwd_out, uint32_t* n_fwd,
                    uint64_t* rc_out, uint32_t* n_rc, uint32_t cap);

/* Seed size the context's index was built with (REF SeedIndex::seed_size, seed_index.hpp:60). */
int sa_index_seed_size(const sa_context* ctx, int32_t* seed_size);

/* Index shape: distinct seeds (REF SeedIndex::distinct_seeds, seed_index.hpp:62),
 * total positions (SeedIndex::total_positions, :61) and device bytes held. */
int sa_index_info(const sa_context* ctx, uint64_t* distinct_seeds,
                  uint64_t* total_positions, uint64_t* device_bytes);

/* bounded_distance over a batch (REF src/edit_distance.cpp:19-75): pair i is
 * read reads[read_off[i]..read_off[i+1]) against window
 * windows[win_off[i]..win_off[i+1]) with limit d_limits[i].  out[i] = the
 * distance or -1 (nullopt).  Runs on `device`.  SA_EINVAL if any d_limit < 0
 * (REF edit_distance.cpp:22-23). */
int sa_bounded_distance_batch(const char* reads, const uint64_t* read_off,
                              const char* windows, const uint64_t* win_off,
                              const int32_t* d_limits, uint64_t n_pairs,
                              int32_t* out, int32_t device);

/* Pinned host memory for zero-staging transfers. */
int sa_host_alloc(void** ptr, uint64_t bytes);
void sa_host_free(void* ptr);

/* Device time (ms, CUDA events) of the last sa_align_batch call from the
 * first H2D copy to the last D2H copy, and of the align kernels alone. */
int sa_last_timing(const sa_context* ctx, float* e2e_ms, float* kernel_ms);

/* Device time (ms, CUDA events) of the last align call's kernels: the fused
 * shared-memory-table kernel and the overflow (global-table) kernel, summed
 * over chunks.  After sa_align_device this waits for those events. */
int sa_last_kernel_times(sa_context* ctx, float* fast_ms, float* slow_ms);

/* Number of CUDA kernels launched by the last sa_align_batch call. */
int sa_last_launches(const sa_context* ctx, uint64_t* launches);

/* ------------------------------------------------------------------ genome and index files
 * sa_genome = PackedGenome (REF include/seedaln/genome.hpp:36-100): packed
 * words, N mask and the contig table. */
typedef struct sa_genome sa_genome;

enum { SA_INDEX_SNAPIDX1 = 0, /* the reference's file, REF include/seedaln/seed_index.hpp:74-85 */
       SA_INDEX_SNAPGPU1 = 1  /* compact: SNAPIDX1 header + genome, no CSR tables (the GPU
                                 rebuilds its index from the genome in seconds) */ };

/* PackedGenome::from_fasta (REF src/genome.cpp:48-94): '>' headers (name =
 * first whitespace-delimited token), IUPAC letters, case and whitespace
 * ignored.  SA_EPARSE with the reference's messages; SA_EIO if unreadable. */
int sa_genome_from_fasta(const char* path, sa_genome** out);

/* A genome from PackedGenome words and its contig table (names[i] NUL-terminated). */
int sa_genome_from_words(const uint64_t* packed, uint64_t n_packed, const uint64_t* nmask, uint64_t n_nmask,
                         uint64_t length, const char* const* names, const uint64_t* starts,
                         const uint64_t* lengths, uint64_t n_contigs, sa_genome** out);
void sa_genome_free(sa_genome* g);

/* size(), contigs().size() and checksum() (REF genome.hpp:59, 91, 95; genome.cpp:158-179). */
int sa_genome_info(const sa_genome* g, uint64_t* length, uint64_t* n_contigs, uint64_t* checksum);
/* packed_words() / n_mask_words() (REF genome.hpp:98-99); pointers valid while g lives. */
int sa_genome_words(const sa_genome* g, const uint64_t** packed, uint64_t* n_packed, const uint64_t** nmask,
                    uint64_t* n_nmask);
/* contigs()[i] (REF genome.hpp:24-28); name valid while g lives. */
int sa_genome_contig(const sa_genome* g, uint64_t i, const char** name, uint64_t* start, uint64_t* length);

/* sa_create over a genome object. */
int sa_create_from_genome(const sa_genome* g, int32_t seed_size, const int32_t* devices, int32_t n_devices,
                          sa_context** out);

/* run_index + save_index_file (REF src/driver.cpp:37-45, src/seed_index.cpp:145-170).
 * SA_INDEX_SNAPIDX1: the CSR tables (REF SeedIndex::build, seed_index.cpp:80-126)
 * are built on GPU `device`; the file is byte-identical to the reference's.
 * SA_INDEX_SNAPGPU1: header + genome only. */
int sa_index_write(const sa_genome* g, int32_t seed_size, int32_t format, int32_t device, const char* path);

/* load_index_file (REF src/seed_index.cpp:173-228) followed by sa_create on
 * `devices`: reads SNAPIDX1 or SNAPGPU1 with the reference's checks and
 * messages (SA_EFORMAT).  With verify != 0 the SNAPIDX1 tables are compared
 * with a GPU rebuild from the embedded genome (SA_EFORMAT on mismatch), since
 * the GPU aligns with its own index of that genome.  The caller frees both. */
int sa_index_load(const char* path, const int32_t* devices, int32_t n_devices, int32_t verify,
                  sa_genome** genome_out, sa_context** ctx_out);

/* The reference's CSR tables of g (SeedIndex keys_/offsets_/positions_, REF
 * include/seedaln/seed_index.hpp:69-71), built on GPU `device`.  On entry
 * *n_keys / *n_positions are the capacities of keys (offsets: n_keys + 1) and
 * positions; on return the sizes.  NULL arrays: sizes only. */
int sa_index_csr(const sa_genome* g, int32_t seed_size, int32_t device, uint64_t* n_keys, uint64_t* n_positions,
                 uint64_t* keys, uint64_t* offsets, uint64_t* positions);

/* ------------------------------------------------------------------ referee
 * The exhaustive referee of the evaluation harness on the GPU: OracleContext,
 * oracle_scan, oracle_align (REF include/seedaln/eval.hpp:49-117,
 * src/eval.cpp:122-306).  Exact; used for accuracy evaluation at scale. */
typedef struct sa_referee sa_referee;

/* OracleHit (REF eval.hpp:93-97). */
typedef struct sa_referee_hit {
    uint64_t position;
    int32_t distance;
    uint8_t direction;
    uint8_t reserved[3];
} sa_referee_hit;

/* OracleContext(g) (REF src/eval.cpp:155-165): genome planes and the q-gram
 * tables (q_hi sized to the genome, then 7, 6, 5) built on `device`. */
int sa_referee_create(const sa_genome* g, int32_t device, sa_referee** out);
void sa_referee_destroy(sa_referee* r);

/* oracle_align (REF src/eval.cpp:270-306) per read: staged limits, the
 * aligner's BestTracker and classify_confidence.  Reads as in sa_align_batch;
 * SA_EINVAL on a character outside {A,C,G,T,N} (REF genome.cpp:194-195). */
int sa_referee_align(sa_referee* r, const sa_params* params, const char* bases, const uint64_t* offsets,
                     uint64_t n_reads, sa_result* results);

/* oracle_scan (REF src/eval.cpp:244-268) per read: read i's hits (best-first,
 * ties by position, Forward first) are hits[hit_offsets[i] .. hit_offsets[i+1]).
 * hit_offsets has n_reads + 1 entries; hits (capacity cap) may be NULL to size. */
int sa_referee_scan(sa_referee* r, int32_t d_limit, int32_t bucket_size, const char* bases,
                    const uint64_t* offsets, uint64_t n_reads, uint64_t* hit_offsets, sa_referee_hit* hits,
                    uint64_t cap);

/* ------------------------------------------------------------------ FASTQ -> SAM driver
 * AlignOptions (REF include/seedaln/driver.hpp:20-32) plus the devices to use. */
typedef struct sa_align_options {
    const char* index_path;    /* SNAPIDX1 or SNAPGPU1 */
    const char* fastq_path;
    const char* output_path;   /* SAM */
    sa_params params;
    uint32_t threads;          /* host workers; 0 = hardware concurrency */
    uint64_t chunk_min_bytes;  /* scheduler minimum chunk (REF scheduler.cpp:8-16) */
    int32_t stable_order;      /* write records in input order */
    uint64_t tolerance;        /* truth-scoring window, bases */
    const char* report_path;   /* optional key=value metrics file (NULL/"" = none) */
    const char* command_line;  /* @PG CL: */
    const int32_t* devices;    /* GPUs (NULL = device 0) */
    int32_t n_devices;
    int32_t verify_index;      /* see sa_index_load */
} sa_align_options;

/* EvalReport (REF include/seedaln/eval.hpp:24-46). */
typedef struct sa_eval_report {
    uint64_t total, single, multiple, notfound, correct, wrong, no_truth;
    double elapsed_seconds;
    sa_stats stats;
} sa_eval_report;

/* AlignOptions{} defaults (REF driver.hpp:20-32). */
void sa_default_align_options(sa_align_options* out);

/* run_index (REF src/driver.cpp:37-45): FASTA -> index file (see sa_index_write). */
int sa_run_index(const char* fasta_path, const char* index_path, int32_t seed_size, int32_t format,
                 int32_t device);

/* run_align (REF src/driver.cpp:47-156): index + FASTQ -> SAM, one record
 * per read (REF src/sam.cpp:11-87), the reference's chunk scheduler over host
 * workers, every chunk's reads aligned on the GPU in one batch, truth scored
 * from read names (REF src/eval.cpp:12-33).  With stable_order the SAM is
 * byte-identical to the reference's.  Errors carry the reference's exception
 * class (SA_EINVAL / SA_EFORMAT / SA_EPARSE / SA_EIO) and message. */
int sa_run_align(const sa_align_options* opt, sa_eval_report* report);

/* EvalReport::to_text (REF src/eval.cpp:75-120) into out (capacity cap, NUL
 * terminated); *len = full length. */
int sa_report_text(const sa_eval_report* r, char* out, uint64_t cap, uint64_t* len);

/* ------------------------------------------------------------------ read simulator
 * SimProfile (REF include/seedaln/simulator.hpp:17-26). */
typedef struct sa_sim_profile {
    uint64_t read_length;
    double snp_rate;
    double indel_mutation_rate;
    double seq_error_rate;
    double indel_error_fraction;
    uint64_t rng_seed;
} sa_sim_profile;

/* Truth (REF simulator.hpp:30-36); contig = index into the genome's contig
 * table; the read name is encode_truth (REF src/simulator.cpp:43-48):
 * "<contig name>_<position+1>_<F|R>_<serial>". */
typedef struct sa_sim_truth {
    uint64_t contig;
    uint64_t position;  /* 0-based offset within the contig */
    uint64_t serial;
    uint8_t direction;  /* SA_FORWARD / SA_REVERSE_COMPLEMENT */
} sa_sim_truth;

typedef struct sa_simulator sa_simulator;

/* SimProfile{} defaults (REF simulator.hpp:17-24). */
void sa_default_sim_profile(sa_sim_profile* out);

/* ReadSimulator(genome, profile) (REF src/simulator.cpp:90-99): validates the
 * profile (SA_EINVAL, SimProfile::validate messages) and that some contig
 * fits a read.  g must outlive the simulator. */
int sa_simulator_create(const sa_genome* g, const sa_sim_profile* p, sa_simulator** out);
void sa_simulator_destroy(sa_simulator* s);

/* `count` calls of ReadSimulator::next (REF src/simulator.cpp:117-192): the
 * same mt19937_64 draw stream, so the reads are the reference's.  bases gets
 * count * read_length chars (the read as Read::bases, reverse-complemented
 * for R reads), truth gets count entries.  SA_ERUNTIME "failed to place a
 * read; genome may be mostly N" after 10,000 redraws (reads before it stay). */
int sa_simulator_next(sa_simulator* s, uint64_t count, char* bases, sa_sim_truth* truth);

/* run_simulate (REF src/driver.cpp:158-168): FASTA -> `count` FASTQ records
 * (to_fastq, REF simulator.cpp:194-206), byte-identical to the reference's
 * file.  Generation is one sequential stream; `threads` host threads (0 =
 * hardware concurrency) format the records while the next batch is drawn. */
int sa_run_simulate(const char* fasta_path, const char* output_path, uint64_t count, const sa_sim_profile* p,
                    uint32_t threads);

#ifdef __cplusplus
}
#endif

#endif /* SNAP_B200_H */
