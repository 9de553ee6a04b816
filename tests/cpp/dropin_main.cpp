// dropin_main.cpp -- TEST PROGRAM (tests/test_boundary.py runs it on a GPU).
//
// The C++ drop-in executed: one process links the UNMODIFIED reference
// library (oracle/_ref/libseedaln_ref.so, compiled from /root/reference) and
// the GPU library through include/snap_b200.hpp, and aligns the same reads
// both ways the way the reference's run_align worker does (REF
// src/driver.cpp:99-132: pageable std::string reads, one Aligner per worker,
// results in read order).  Every AlignmentResult field and the AlignStats
// counters are compared; the exception contract is checked too.
// Prints "DROPIN OK <reads> <mismatches>" and exits 0 when all agree.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "seedaln/aligner.hpp"
#include "seedaln/genome.hpp"
#include "seedaln/read.hpp"
#include "seedaln/seed_index.hpp"
#include "snap_b200.hpp"

namespace {

std::string make_genome(uint64_t len, uint64_t seed) {
    // i.i.d. background with planted diverged repeat copies, so reads hit
    // several loci (multi-hit seeds, many candidates, popular seeds)
    std::mt19937_64 rng(seed);
    std::string g(len, 'A');
    for (auto& c : g) c = "ACGT"[rng() % 4];
    for (int fam = 0; fam < 40; ++fam) {
        const uint64_t L = 200 + rng() % 1200;
        const uint64_t src = rng() % (len - L);
        const std::string cons = g.substr(src, L);
        const int copies = 2 + static_cast<int>(rng() % 60);
        for (int k = 0; k < copies; ++k) {
            const uint64_t dst = rng() % (len - L);
            for (uint64_t i = 0; i < L; ++i)
                g[dst + i] = (rng() % 100 < 3) ? "ACGT"[rng() % 4] : cons[i];
        }
    }
    for (int r = 0; r < 20; ++r) {  // N runs
        const uint64_t p = rng() % (len - 50);
        for (uint64_t i = 0, n = 1 + rng() % 30; i < n; ++i) g[p + i] = 'N';
    }
    return g;
}

std::vector<seedaln::Read> make_reads(const std::string& g, size_t n, uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::vector<seedaln::Read> reads(n);
    auto comp = [](char c) { return c == 'A' ? 'T' : c == 'C' ? 'G' : c == 'G' ? 'C' : c == 'T' ? 'A' : 'N'; };
    for (size_t i = 0; i < n; ++i) {
        const uint64_t L = (i % 97 == 0) ? 10 + rng() % 200 : 100 + rng() % 51;  // ragged, a few short
        const uint64_t p = rng() % (g.size() - L);
        std::string b = g.substr(p, L);
        for (auto& c : b)
            if (rng() % 100 < 2) c = "ACGT"[rng() % 4];
        if (rng() % 2) {
            std::string rc(b.rbegin(), b.rend());
            for (auto& c : rc) c = comp(c);
            b = rc;
        }
        if (i % 53 == 0) b[rng() % b.size()] = 'N';
        reads[i].name = "r" + std::to_string(i);
        reads[i].bases = b;
        reads[i].qualities.assign(b.size(), 'I');
    }
    return reads;
}

int expect_invalid(const char* what, auto&& fn) {
    try {
        fn();
    } catch (const std::invalid_argument&) {
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s: wrong exception type: %s\n", what, e.what());
        return 1;
    }
    std::fprintf(stderr, "%s: no exception\n", what);
    return 1;
}

}  // namespace

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 200000;
    const std::string seq = make_genome(4'000'000, 11);
    const seedaln::PackedGenome genome = seedaln::PackedGenome::from_contigs({{"chr1", seq}});
    const std::vector<seedaln::Read> reads = make_reads(seq, n, 12);
    int fails = 0;
    size_t total = 0, bad = 0;
    for (int variant = 0; variant < 3; ++variant) {
        seedaln::AlignerParams rp;
        rp.seeds_to_try = variant == 1 ? 14 : 10;
        rp.max_hits = variant == 2 ? 40 : 300;
        rp.bucket_size = variant == 2 ? 16 : 32;
        // the reference worker: one Aligner, read by read (REF src/driver.cpp:102-113)
        const seedaln::SeedIndex ridx = seedaln::SeedIndex::build(genome, rp.seed_size);
        seedaln::Aligner ref(ridx, genome, rp);
        std::vector<seedaln::AlignmentResult> want;
        want.reserve(reads.size());
        for (const auto& r : reads) want.push_back(ref.align(r));
        // the drop-in: the same genome words, the same params, one batch
        snap_b200::SeedIndex gidx(genome.packed_words(), genome.n_mask_words(), genome.size(), rp.seed_size);
        sa_params gp = snap_b200::default_params();
        gp.seed_size = rp.seed_size;
        gp.seeds_to_try = rp.seeds_to_try;
        gp.max_distance = rp.max_distance;
        gp.confidence_threshold = rp.confidence_threshold;
        gp.max_hits = rp.max_hits;
        gp.bucket_size = rp.bucket_size;
        gp.force_max_dlimit = rp.force_max_dlimit ? 1 : 0;
        snap_b200::Aligner al(gidx, gp);
        const std::vector<sa_result> got = al.align_reads(reads);
        for (size_t i = 0; i < reads.size(); ++i) {
            const auto& w = want[i];
            const auto& g = got[i];
            const bool same = g.kind == static_cast<uint8_t>(w.kind) && g.has_position == (w.has_position ? 1 : 0) &&
                              g.position == w.position && g.direction == static_cast<uint8_t>(w.direction) &&
                              g.distance == w.distance && g.gap == w.gap;
            if (!same && bad++ < 5)
                std::fprintf(stderr, "variant %d read %zu: gpu kind %d pos %llu dir %d d %d gap %d | ref kind %d pos %llu dir %d d %d gap %d\n",
                             variant, i, g.kind, (unsigned long long)g.position, g.direction, g.distance, g.gap,
                             (int)w.kind, (unsigned long long)w.position, (int)w.direction, w.distance, w.gap);
        }
        total += reads.size();
        const auto& rs = ref.stats();
        const auto& gs = al.stats();
        const uint64_t pairs[][2] = {{rs.reads, gs.reads}, {rs.reads_too_short, gs.reads_too_short},
                                     {rs.seed_lookups, gs.seed_lookups}, {rs.seeds_skipped_n, gs.seeds_skipped_n},
                                     {rs.seeds_skipped_popular, gs.seeds_skipped_popular},
                                     {rs.reads_all_seeds_popular, gs.reads_all_seeds_popular},
                                     {rs.distance_calls, gs.distance_calls},
                                     {rs.distance_calls_after_first, gs.distance_calls_after_first},
                                     {rs.early_out_after_first, gs.early_out_after_first},
                                     {rs.multi_early_exits, gs.multi_early_exits}, {rs.pruning_exits, gs.pruning_exits},
                                     {rs.first_scored_was_best, gs.first_scored_was_best},
                                     {rs.single_hits, gs.single_hits}, {rs.multiple_hits, gs.multiple_hits},
                                     {rs.not_found, gs.not_found}};
        for (size_t k = 0; k < sizeof(pairs) / sizeof(pairs[0]); ++k)
            if (pairs[k][0] != pairs[k][1]) {
                std::fprintf(stderr, "variant %d stat %zu: ref %llu gpu %llu\n", variant, k,
                             (unsigned long long)pairs[k][0], (unsigned long long)pairs[k][1]);
                ++fails;
            }
        // single-read call (REF Aligner::align shape)
        const sa_result one = al.align(reads[1].bases);
        if (one.kind != static_cast<uint8_t>(want[1].kind) || one.position != want[1].position) ++fails;
    }
    // exception contract (REF aligner.cpp:11-24,116-122; genome.cpp:182-200)
    snap_b200::SeedIndex gidx(genome.packed_words(), genome.n_mask_words(), genome.size(), 20);
    fails += expect_invalid("bucket_size 0", [&] {
        sa_params p = snap_b200::default_params();
        p.bucket_size = 0;
        snap_b200::Aligner a(gidx, p);
    });
    fails += expect_invalid("seed size mismatch", [&] {
        sa_params p = snap_b200::default_params();
        p.seed_size = 22;
        snap_b200::Aligner a(gidx, p);
    });
    fails += expect_invalid("bad character", [&] {
        snap_b200::Aligner a(gidx, snap_b200::default_params());
        std::vector<seedaln::Read> rr(2);
        rr[0].bases = reads[0].bases;
        rr[1].bases = std::string(120, 'A') + "X";
        a.align_reads(rr);
    });
    fails += expect_invalid("reference bad character", [&] {
        seedaln::AlignerParams rp;
        const seedaln::SeedIndex ridx = seedaln::SeedIndex::build(genome, 20);
        seedaln::Aligner ref(ridx, genome, rp);
        seedaln::Read r;
        r.bases = std::string(120, 'A') + "X";
        ref.align(r);
    });
    std::printf("DROPIN %s %zu %zu\n", (bad == 0 && fails == 0) ? "OK" : "FAIL", total, bad);
    return (bad == 0 && fails == 0) ? 0 : 1;
}
