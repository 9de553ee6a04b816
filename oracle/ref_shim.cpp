// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" harness around the UNMODIFIED reference library
// (/root/reference/proj/src, compiled in place by oracle/Makefile into
// oracle/_ref/libseedaln_ref.so).  It calls only the reference's public API:
//   PackedGenome::adopt_storage  (REF include/seedaln/genome.hpp:75-76)
//   SeedIndex::build / lookup    (REF src/seed_index.cpp:80-143)
//   bounded_distance / full_dp   (REF src/edit_distance.cpp:19-95)
//   seed_offsets / Aligner::align(REF src/aligner.cpp:50-79,223-364)
//   PackedGenome::from_fasta, save/load_index_file, run_index, run_align
//                                (REF src/genome.cpp, seed_index.cpp:145-228, driver.cpp)
// and the align_corpus threading pattern of the acceptance suite
// (REF tests/acceptance/acceptance_main.cpp:52-67,106-124).
// Used by tests/ as the parity pin for the C restatement, and by bench.py's
// cpu_baseline and --impl reference legs.  Never part of the product.
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../include/snap_b200.h"
#include <fstream>
#include <istream>
#include <streambuf>

#include "seedaln/aligner.hpp"
#include "seedaln/driver.hpp"
#include "seedaln/edit_distance.hpp"
#include "seedaln/errors.hpp"
#include "seedaln/eval.hpp"
#include "seedaln/genome.hpp"
#include "seedaln/seed_index.hpp"

using namespace seedaln;

namespace {

struct RefHandle {
    PackedGenome genome;
    SeedIndex index;
};

thread_local std::string g_err;

void fill_stats(const AlignStats& a, sa_stats* out) {
    uint64_t* d = reinterpret_cast<uint64_t*>(out);
    const uint64_t v[16] = {a.reads,
                            a.reads_too_short,
                            a.seed_lookups,
                            a.seeds_skipped_n,
                            a.seeds_skipped_popular,
                            a.reads_all_seeds_popular,
                            a.distance_calls,
                            a.distance_calls_after_first,
                            a.early_out_after_first,
                            a.dp_cells,
                            a.multi_early_exits,
                            a.pruning_exits,
                            a.first_scored_was_best,
                            a.single_hits,
                            a.multiple_hits,
                            a.not_found};
    for (int i = 0; i < 16; ++i) d[i] += v[i];
}

AlignerParams to_params(const sa_params* p) {
    AlignerParams a;
    a.seed_size = p->seed_size;
    a.seeds_to_try = p->seeds_to_try;
    a.max_distance = p->max_distance;
    a.confidence_threshold = p->confidence_threshold;
    a.max_hits = p->max_hits;
    a.bucket_size = p->bucket_size;
    a.force_max_dlimit = p->force_max_dlimit != 0;
    return a;
}

void to_result(const AlignmentResult& r, sa_result* out) {
    std::memset(out, 0, sizeof(*out));
    out->position = r.position;
    out->distance = r.distance;
    out->gap = r.gap;
    out->kind = static_cast<uint8_t>(r.kind);
    out->has_position = r.has_position ? 1 : 0;
    out->direction = static_cast<uint8_t>(r.direction);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_create(const uint64_t* packed, uint64_t n_packed, const uint64_t* nmask,
                 uint64_t n_nmask, uint64_t len, int seed_size) {
    try {
        auto* h = new RefHandle;
        std::vector<Contig> contigs{{"c1", 0, len}};
        h->genome.adopt_storage(std::move(contigs), len,
                                std::vector<uint64_t>(packed, packed + n_packed),
                                std::vector<uint64_t>(nmask, nmask + n_nmask));
        h->index = SeedIndex::build(h->genome, seed_size);
        return h;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// The reference's SeedIndex over a key-restricted CSR (keys ascending in the
// reference's packed form, CSR offsets, u32 positions ascending per key), as
// the oracle's or_index_build_for_reads makes for a batch of reads.  The
// tables go through the reference's own load_index_file (REF
// src/seed_index.cpp:173-228, all its checks) from an in-memory SNAPIDX1
// image, so the reference's unmodified lookup and Aligner run on them.  For
// every key those reads probe the answer equals SeedIndex::build's; this is
// how the reference arm runs at 3.1 Gbp, where the full single-threaded build
// (REF seed_index.cpp:80-126, ~115 GB peak) does not fit a bounded run.
void* ref_create_from_csr(const uint64_t* packed, uint64_t n_packed, const uint64_t* nmask, uint64_t n_nmask,
                          uint64_t len, int seed_size, const uint64_t* keys, uint64_t n_keys,
                          const uint64_t* offsets, const uint32_t* positions, uint64_t n_pos) {
    try {
        PackedGenome g;
        std::vector<Contig> contigs{{"c1", 0, len}};
        g.adopt_storage(std::move(contigs), len, std::vector<uint64_t>(packed, packed + n_packed),
                        std::vector<uint64_t>(nmask, nmask + n_nmask));
        const uint64_t sum = g.checksum();
        std::vector<char> img;
        img.reserve(64 + 8 * (n_packed + n_nmask + 2 * n_keys + n_pos + 8));
        auto put = [&](const void* p, size_t n) {
            const char* c = static_cast<const char*>(p);
            img.insert(img.end(), c, c + n);
        };
        auto u32 = [&](uint32_t v) { put(&v, 4); };  // little-endian host (x86-64)
        auto u64 = [&](uint64_t v) { put(&v, 8); };
        put("SNAPIDX1", 8);
        u32(1);
        u32(static_cast<uint32_t>(seed_size));
        u64(sum);
        u64(1);
        u32(2);
        put("c1", 2);
        u64(0);
        u64(len);
        u64(len);
        u64(n_packed);
        put(packed, 8 * n_packed);
        u64(n_nmask);
        put(nmask, 8 * n_nmask);
        u64(n_keys);
        put(keys, 8 * n_keys);
        u64(n_keys + 1);
        put(offsets, 8 * (n_keys + 1));
        u64(n_pos);
        for (uint64_t i = 0; i < n_pos; ++i) u64(positions[i]);
        put("SNAPEND1", 8);
        struct MemBuf : std::streambuf {
            MemBuf(char* b, size_t n) { setg(b, b, b + n); }
        } mb(img.data(), img.size());
        std::istream in(&mb);
        auto loaded = load_index_file(in);
        auto* h = new RefHandle;
        h->index = std::move(loaded.first);
        h->genome = std::move(loaded.second);
        return h;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_destroy(void* h) { delete static_cast<RefHandle*>(h); }

void ref_index_info(void* hv, uint64_t* distinct, uint64_t* total) {
    auto* h = static_cast<RefHandle*>(hv);
    *distinct = h->index.distinct_seeds();
    *total = h->index.total_positions();
}

uint64_t ref_genome_checksum(void* hv) { return static_cast<RefHandle*>(hv)->genome.checksum(); }

// returns 0 ok, 1 invalid_argument
int ref_lookup(void* hv, const char* seed, int s, uint64_t* fwd, uint64_t* n_fwd, uint64_t* rc,
               uint64_t* n_rc, uint64_t cap) {
    auto* h = static_cast<RefHandle*>(hv);
    try {
        LookupResult r = h->index.lookup(std::string_view(seed, static_cast<size_t>(s)));
        *n_fwd = r.forward.size();
        *n_rc = r.rc.size();
        for (size_t i = 0; i < r.forward.size() && i < cap; ++i) fwd[i] = r.forward[i];
        for (size_t i = 0; i < r.rc.size() && i < cap; ++i) rc[i] = r.rc[i];
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// -1 = nullopt, -2 = threw invalid_argument
int ref_bounded_distance(const char* read, uint64_t m, const char* win, uint64_t w, int d_limit,
                         uint64_t* cells) {
    try {
        DistanceOutcome o = bounded_distance(std::string_view(read, m), std::string_view(win, w),
                                             d_limit, cells);
        return o ? *o : -1;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -2;
    }
}

int ref_full_dp_distance(const char* read, uint64_t m, const char* win, uint64_t w) {
    return full_dp_distance(std::string_view(read, m), std::string_view(win, w));
}

int ref_seed_offsets(uint64_t len, int s, int n, int* out) {
    std::vector<int> v = seed_offsets(len, s, n);
    for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
    return static_cast<int>(v.size());
}

int ref_pack_seed(const char* seed, int s, uint64_t* out) {
    return pack_seed(std::string_view(seed, static_cast<size_t>(s)), *out) ? 1 : 0;
}

uint64_t ref_packed_rc(uint64_t key, int s) { return packed_reverse_complement(key, s); }

// BestTracker replay for known-answer tests: ops = (distance, position, dir)
// triples; writes (d_best, d_second, best_position, gap) after each op.
void ref_tracker_replay(int merge_radius, const int64_t* ops, int n_ops, int64_t* out) {
    BestTracker t(merge_radius);
    for (int i = 0; i < n_ops; ++i) {
        t.observe(static_cast<int>(ops[3 * i]), static_cast<uint64_t>(ops[3 * i + 1]),
                  static_cast<Direction>(ops[3 * i + 2]));
        out[4 * i] = t.d_best();
        out[4 * i + 1] = t.d_second();
        out[4 * i + 2] = static_cast<int64_t>(t.best_position());
        out[4 * i + 3] = t.gap();
    }
}

// 0 ok, 1 invalid_argument (params, or a read the reference rejects)
int ref_align_batch(void* hv, const sa_params* p, const char* bases, const uint64_t* offsets,
                    uint64_t n, sa_result* results, sa_stats* stats, int threads) {
    auto* h = static_cast<RefHandle*>(hv);
    AlignerParams params = to_params(p);
    try {
        params.validate();
        Aligner probe(h->index, h->genome, params);  // throws on seed-size mismatch
        (void)probe;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
    if (threads < 1) threads = 1;
    std::atomic<uint64_t> cursor{0};
    std::atomic<bool> failed{false};
    std::mutex mu;
    AlignStats total;
    auto body = [&]() {
        Aligner local(h->index, h->genome, params);
        try {
            const uint64_t grain = 64;
            while (!failed.load()) {
                uint64_t begin = cursor.fetch_add(grain);
                if (begin >= n) break;
                uint64_t end = std::min(n, begin + grain);
                for (uint64_t i = begin; i < end; ++i) {
                    Read r;
                    r.bases.assign(bases + offsets[i], offsets[i + 1] - offsets[i]);
                    to_result(local.align(r), &results[i]);
                }
            }
        } catch (const std::exception& e) {
            std::lock_guard<std::mutex> lock(mu);
            g_err = e.what();
            failed = true;
        }
        std::lock_guard<std::mutex> lock(mu);
        total.merge(local.stats());
    };
    if (threads == 1) {
        body();
    } else {
        std::vector<std::thread> th;
        for (int t = 0; t < threads; ++t) th.emplace_back(body);
        for (auto& t : th) t.join();
    }
    if (stats) fill_stats(total, stats);
    return failed ? 1 : 0;
}


// ---------------------------------------------------------------- files

// exception class -> sa status code (include/snap_b200.h)
static int code_of(const std::exception_ptr& ep) {
    try {
        std::rethrow_exception(ep);
    } catch (const ParseError& e) {
        g_err = e.what();
        return 4;
    } catch (const FormatError& e) {
        g_err = e.what();
        return 3;
    } catch (const IoError& e) {
        g_err = e.what();
        return 5;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

struct RefGenome {
    PackedGenome g;
};

int ref_genome_from_fasta(const char* path, void** out) {
    try {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw IoError(std::string("cannot open ") + path + " for reading");
        auto* h = new RefGenome{PackedGenome::from_fasta(in)};
        *out = h;
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

void ref_genome_free(void* h) { delete static_cast<RefGenome*>(h); }

void ref_genome_info(void* hv, uint64_t* len, uint64_t* n_contigs, uint64_t* checksum) {
    const PackedGenome& g = static_cast<RefGenome*>(hv)->g;
    *len = g.size();
    *n_contigs = g.contigs().size();
    *checksum = g.checksum();
}

void ref_genome_words(void* hv, const uint64_t** packed, uint64_t* n_packed, const uint64_t** nmask,
                      uint64_t* n_nmask) {
    const PackedGenome& g = static_cast<RefGenome*>(hv)->g;
    *packed = g.packed_words().data();
    *n_packed = g.packed_words().size();
    *nmask = g.n_mask_words().data();
    *n_nmask = g.n_mask_words().size();
}

void ref_genome_contig(void* hv, uint64_t i, const char** name, uint64_t* start, uint64_t* len) {
    const Contig& c = static_cast<RefGenome*>(hv)->g.contigs()[i];
    *name = c.name.c_str();
    *start = c.start;
    *len = c.length;
}

// run_index (REF src/driver.cpp:37-45)
int ref_run_index(const char* fasta, const char* index_path, int seed_size) {
    try {
        IndexOptions o;
        o.fasta_path = fasta;
        o.index_path = index_path;
        o.seed_size = seed_size;
        run_index(o);
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}

// load_index_file (REF src/seed_index.cpp:173-228) -> a handle usable with
// ref_align_batch / ref_lookup
int ref_load_index(const char* path, void** out) {
    try {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw IoError(std::string("cannot open ") + path + " for reading");
        auto [idx, g] = load_index_file(in);
        auto* h = new RefHandle;
        h->genome = std::move(g);
        h->index = std::move(idx);
        *out = h;
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}


// run_simulate (REF src/driver.cpp:158-168) with a SimProfile
int ref_run_simulate(const char* fasta, const char* out_path, uint64_t count, uint64_t read_length,
                     double snp_rate, double indel_mutation_rate, double seq_error_rate,
                     double indel_error_fraction, uint64_t rng_seed) {
    try {
        SimulateOptions o;
        o.fasta_path = fasta;
        o.output_path = out_path;
        o.count = count;
        o.profile.read_length = read_length;
        o.profile.snp_rate = snp_rate;
        o.profile.indel_mutation_rate = indel_mutation_rate;
        o.profile.seq_error_rate = seq_error_rate;
        o.profile.indel_error_fraction = indel_error_fraction;
        o.profile.rng_seed = rng_seed;
        run_simulate(o);
        return 0;
    } catch (...) {
        return code_of(std::current_exception());
    }
}



// ---------------------------------------------------------------- referee

struct RefReferee {
    PackedGenome g;
    std::unique_ptr<OracleContext> ctx;
};

// OracleContext over a one-contig genome (REF src/eval.cpp:155-165)
void* ref_referee_create(const uint64_t* packed, uint64_t n_packed, const uint64_t* nmask, uint64_t n_nmask,
                         uint64_t len) {
    try {
        auto* h = new RefReferee;
        std::vector<Contig> contigs{{"c1", 0, len}};
        h->g.adopt_storage(std::move(contigs), len, std::vector<uint64_t>(packed, packed + n_packed),
                           std::vector<uint64_t>(nmask, nmask + n_nmask));
        h->ctx = std::make_unique<OracleContext>(h->g);
        return h;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_referee_destroy(void* h) { delete static_cast<RefReferee*>(h); }

// oracle_align (REF src/eval.cpp:270-306) over a batch, `threads` workers
int ref_oracle_align(void* hv, const sa_params* p, const char* bases, const uint64_t* offsets, uint64_t n,
                     sa_result* results, int threads) {
    auto* h = static_cast<RefReferee*>(hv);
    AlignerParams prm;
    prm.seed_size = p->seed_size;
    prm.seeds_to_try = p->seeds_to_try;
    prm.max_distance = p->max_distance;
    prm.confidence_threshold = p->confidence_threshold;
    prm.max_hits = p->max_hits;
    prm.bucket_size = p->bucket_size;
    std::atomic<uint64_t> cursor{0};
    std::atomic<bool> failed{false};
    std::mutex mu;
    auto body = [&]() {
        try {
            for (;;) {
                uint64_t i = cursor.fetch_add(1);
                if (i >= n || failed.load()) break;
                Read r;
                r.bases.assign(bases + offsets[i], offsets[i + 1] - offsets[i]);
                to_result(oracle_align(r, *h->ctx, prm), &results[i]);
            }
        } catch (const std::exception& e) {
            std::lock_guard<std::mutex> lock(mu);
            g_err = e.what();
            failed = true;
        }
    };
    std::vector<std::thread> th;
    for (int t = 0; t < std::max(1, threads); ++t) th.emplace_back(body);
    for (auto& t : th) t.join();
    return failed ? 1 : 0;
}

// oracle_scan (REF src/eval.cpp:244-268) of one read: hits into out (cap),
// returns the hit count or -1 on error
int64_t ref_oracle_scan(void* hv, const char* read, uint64_t len, int d_limit, int bucket, uint64_t* pos,
                        int32_t* dist, uint8_t* dir, uint64_t cap) {
    try {
        auto* h = static_cast<RefReferee*>(hv);
        Read r;
        r.bases.assign(read, len);
        std::vector<OracleHit> hits = oracle_scan(r, *h->ctx, d_limit, bucket);
        for (size_t i = 0; i < hits.size() && i < cap; ++i) {
            pos[i] = hits[i].position;
            dist[i] = hits[i].distance;
            dir[i] = static_cast<uint8_t>(hits[i].direction);
        }
        return static_cast<int64_t>(hits.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
