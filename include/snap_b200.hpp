// snap_b200.hpp -- header-only C++ adapter over the C ABI (snap_b200.h) that
// restores the reference's C++ shape and exception contract:
//
//   seedaln::SeedIndex::build(genome, s)        -> snap_b200::SeedIndex(packed, nmask, len, s)
//   seedaln::Aligner(idx, genome, params)       -> snap_b200::Aligner(idx, params)
//   Aligner::align(const Read&)                 -> Aligner::align(std::string_view)   (batch of 1; tests)
//                                               -> Aligner::align_batch(...)          (production)
//   PackedGenome::from_fasta                    -> snap_b200::Genome::from_fasta
//   run_index / save_index_file                 -> snap_b200::run_index / save_index_file
//   load_index_file                             -> snap_b200::load_index_file
//   run_align (FASTQ -> SAM)                    -> snap_b200::run_align
//   ReadSimulator / run_simulate               -> snap_b200::ReadSimulator / run_simulate
//   OracleContext / oracle_align / oracle_scan  -> snap_b200::Referee
//   std::invalid_argument / FormatError / ParseError / IoError are rethrown
//   from the status codes (REF include/seedaln/errors.hpp:10-30).
//
// Link with paper_1111_5572_b200/lib/libsnapb200.so.  See INTEGRATION.md.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "snap_b200.h"

namespace snap_b200 {

class FormatError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class ParseError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class IoError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

inline void check(int rc, const sa_context* ctx) {
    if (rc == SA_OK) return;
    std::string msg = sa_last_error(ctx);
    if (rc == SA_EINVAL) throw std::invalid_argument(msg);
    if (rc == SA_EFORMAT) throw FormatError(msg);
    if (rc == SA_EPARSE) throw ParseError(msg);
    if (rc == SA_EIO) throw IoError(msg);
    throw std::runtime_error(msg);
}

inline sa_params default_params() {
    sa_params p;
    sa_default_params(&p);
    return p;
}

// Seed index + genome replica(s) resident in HBM (replaces SeedIndex::build,
// REF src/seed_index.cpp:80-126).  Non-copyable, movable.
class SeedIndex {
public:
    SeedIndex(const std::vector<uint64_t>& packed_words, const std::vector<uint64_t>& n_mask_words,
              uint64_t genome_length, int seed_size, const std::vector<int32_t>& devices = {0}) {
        check(sa_create(packed_words.data(), packed_words.size(), n_mask_words.data(),
                        n_mask_words.size(), genome_length, seed_size, devices.data(),
                        static_cast<int32_t>(devices.size()), &ctx_),
              nullptr);
        seed_size_ = seed_size;
    }
    // adopt a context made elsewhere (load_index_file)
    SeedIndex(sa_context* ctx, int seed_size) : ctx_(ctx), seed_size_(seed_size) {}
    SeedIndex(const SeedIndex&) = delete;
    SeedIndex& operator=(const SeedIndex&) = delete;
    SeedIndex(SeedIndex&& o) noexcept : ctx_(o.ctx_), seed_size_(o.seed_size_) { o.ctx_ = nullptr; }
    ~SeedIndex() { sa_destroy(ctx_); }

    int seed_size() const { return seed_size_; }
    uint64_t distinct_seeds() const {
        uint64_t d = 0;
        check(sa_index_info(ctx_, &d, nullptr, nullptr), ctx_);
        return d;
    }
    uint64_t total_positions() const {
        uint64_t t = 0;
        check(sa_index_info(ctx_, nullptr, &t, nullptr), ctx_);
        return t;
    }
    sa_context* context() const { return ctx_; }

private:
    sa_context* ctx_ = nullptr;
    int seed_size_ = 0;
};

// Replaces seedaln::Aligner (REF include/seedaln/aligner.hpp:116-158).
class Aligner {
public:
    Aligner(const SeedIndex& idx, const sa_params& params) : idx_(&idx), params_(params) {
        check(sa_validate_params(&params_), nullptr);  // REF aligner.cpp:119
        if (idx.seed_size() != params_.seed_size)      // REF aligner.cpp:120-121
            throw std::invalid_argument("index seed size does not match params");
    }

    // reads: bases[offsets[i] .. offsets[i+1]); results in input order
    void align_batch(const char* bases, const uint64_t* offsets, uint64_t n, sa_result* results) {
        sa_stats st{};
        check(sa_align_batch(idx_->context(), &params_, bases, offsets, n, results, &st),
              idx_->context());
        merge(st);
    }

    std::vector<sa_result> align_batch(const std::vector<std::string>& reads) {
        std::string buf;
        std::vector<uint64_t> offs{0};
        for (const auto& r : reads) {
            buf += r;
            offs.push_back(buf.size());
        }
        std::vector<sa_result> out(reads.size());
        align_batch(buf.data(), offs.data(), reads.size(), out.data());
        return out;
    }

    // The run_align worker's batch (REF src/driver.cpp:104-124): any
    // container of Read-like records with a `bases` string (seedaln::Read,
    // REF include/seedaln/read.hpp:9-14).  The bases are gathered into one
    // host buffer; the library packs it into its own pinned buffers.
    template <class Reads, class = decltype(std::declval<const Reads&>().begin()->bases)>
    std::vector<sa_result> align_reads(const Reads& reads) {
        std::string buf;
        std::vector<uint64_t> offs{0};
        for (const auto& r : reads) {
            buf.append(r.bases);
            offs.push_back(buf.size());
        }
        std::vector<sa_result> out(offs.size() - 1);
        if (!out.empty()) align_batch(buf.data(), offs.data(), out.size(), out.data());
        return out;
    }

    sa_result align(std::string_view bases) {  // REF aligner.cpp:223 (batch of one)
        uint64_t offs[2] = {0, bases.size()};
        sa_result r{};
        align_batch(bases.data(), offs, 1, &r);
        return r;
    }

    const sa_stats& stats() const { return stats_; }

private:
    void merge(const sa_stats& s) {  // REF aligner.cpp:31-48
        auto* d = reinterpret_cast<uint64_t*>(&stats_);
        const auto* v = reinterpret_cast<const uint64_t*>(&s);
        for (size_t i = 0; i < sizeof(sa_stats) / sizeof(uint64_t); ++i) d[i] += v[i];
    }

    const SeedIndex* idx_;
    sa_params params_;
    sa_stats stats_{};
};

// PackedGenome with its contig table (REF include/seedaln/genome.hpp:36-100).
class Genome {
public:
    static Genome from_fasta(const std::string& path) {  // REF src/genome.cpp:48-94
        sa_genome* g = nullptr;
        check(sa_genome_from_fasta(path.c_str(), &g), nullptr);
        return Genome(g);
    }
    explicit Genome(sa_genome* g) : g_(g) {}
    Genome(const Genome&) = delete;
    Genome& operator=(const Genome&) = delete;
    Genome(Genome&& o) noexcept : g_(o.g_) { o.g_ = nullptr; }
    ~Genome() { sa_genome_free(g_); }
    uint64_t size() const {
        uint64_t n = 0;
        check(sa_genome_info(g_, &n, nullptr, nullptr), nullptr);
        return n;
    }
    uint64_t checksum() const {
        uint64_t c = 0;
        check(sa_genome_info(g_, nullptr, nullptr, &c), nullptr);
        return c;
    }
    const sa_genome* get() const { return g_; }

private:
    sa_genome* g_ = nullptr;
};

// save_index_file (REF src/seed_index.cpp:145-170), CSR built on the GPU
inline void save_index_file(const Genome& g, int seed_size, const std::string& path,
                            int format = SA_INDEX_SNAPIDX1, int device = 0) {
    check(sa_index_write(g.get(), seed_size, format, device, path.c_str()), nullptr);
}

// run_index (REF src/driver.cpp:37-45)
inline void run_index(const std::string& fasta, const std::string& index_path, int seed_size = 20,
                      int format = SA_INDEX_SNAPIDX1, int device = 0) {
    check(sa_run_index(fasta.c_str(), index_path.c_str(), seed_size, format, device), nullptr);
}

// load_index_file (REF src/seed_index.cpp:173-228) -> (GPU index, genome)
inline std::pair<SeedIndex, Genome> load_index_file(const std::string& path, const std::vector<int32_t>& devices = {0},
                                                    bool verify = true) {
    sa_genome* g = nullptr;
    sa_context* ctx = nullptr;
    check(sa_index_load(path.c_str(), devices.data(), static_cast<int32_t>(devices.size()), verify ? 1 : 0, &g, &ctx),
          nullptr);
    int32_t s = 0;
    sa_index_seed_size(ctx, &s);
    return {SeedIndex(ctx, s), Genome(g)};
}

// run_align (REF src/driver.cpp:47-156): options as AlignOptions
inline sa_eval_report run_align(const sa_align_options& opt) {
    sa_eval_report r{};
    check(sa_run_align(&opt, &r), nullptr);
    return r;
}

// OracleContext + oracle_align / oracle_scan on the GPU (REF src/eval.cpp:155-306)
class Referee {
public:
    explicit Referee(const Genome& g, int device = 0) { check(sa_referee_create(g.get(), device, &r_), nullptr); }
    Referee(const Referee&) = delete;
    Referee& operator=(const Referee&) = delete;
    ~Referee() { sa_referee_destroy(r_); }
    void align_batch(const sa_params& p, const char* bases, const uint64_t* offsets, uint64_t n, sa_result* out) {
        check(sa_referee_align(r_, &p, bases, offsets, n, out), nullptr);
    }

private:
    sa_referee* r_ = nullptr;
};

// ReadSimulator (REF include/seedaln/simulator.hpp:48-66): the reference's reads, in order.
class ReadSimulator {
public:
    ReadSimulator(const Genome& g, const sa_sim_profile& p) : len_(p.read_length) {
        check(sa_simulator_create(g.get(), &p, &s_), nullptr);
    }
    ReadSimulator(const ReadSimulator&) = delete;
    ReadSimulator& operator=(const ReadSimulator&) = delete;
    ~ReadSimulator() { sa_simulator_destroy(s_); }
    // n reads: bases (n * read_length chars) and truths
    void next(uint64_t n, std::string& bases, std::vector<sa_sim_truth>& truth) {
        bases.resize(n * len_);
        truth.resize(n);
        check(sa_simulator_next(s_, n, bases.data(), truth.data()), nullptr);
    }

private:
    sa_simulator* s_ = nullptr;
    uint64_t len_;
};

// run_simulate (REF src/driver.cpp:158-168)
inline void run_simulate(const std::string& fasta, const std::string& out, uint64_t count, const sa_sim_profile& p,
                         uint32_t threads = 0) {
    check(sa_run_simulate(fasta.c_str(), out.c_str(), count, &p, threads), nullptr);
}

}  // namespace snap_b200
