// synth.cpp -- deterministic synthetic genomes and reads for configs C0..C4.
//
// BASELINE.json names no public dataset; these seeded generators stand in for
// the paper's hg19/wgsim inputs.  Input
// generation only: not on the aligner hot path.
//
//  * random genome: chunk c of 2^26 bases draws "ACGT"[rng() % 4] from
//    mt19937_64(c == 0 ? seed : splitmix64(seed + c)).  For genomes up to
//    64 Mbp this is exactly fixtures::random_sequence(seed, len)
//    (REF tests/acceptance/fixtures.cpp:28-35).
//  * repeat genome (C2/C3): random background, then repeat families planted
//    by overwrite at uniform positions (see synth_repeat_genome).
//  * reads: per-read xoshiro256** stream seeded from (seed, read index); start
//    uniform, strand 50/50, per template base an indel event with probability
//    indel_rate (length Geometric(p) clamped to max_indel, insertion or
//    deletion 50/50), else a substitution with probability sub_rate.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

namespace {

inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

struct Xoshiro {
    uint64_t s[4];
    explicit Xoshiro(uint64_t seed) {
        uint64_t x = seed;
        for (int i = 0; i < 4; ++i) {
            x += 0x9E3779B97F4A7C15ull;
            s[i] = splitmix64(x);
        }
    }
    static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    inline uint64_t operator()() {
        uint64_t r = rotl(s[1] * 5, 7) * 9;
        uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl(s[3], 45);
        return r;
    }
    inline double unit() { return static_cast<double>((*this)() >> 11) * 0x1.0p-53; }
};

constexpr char kAcgt[4] = {'A', 'C', 'G', 'T'};

inline char comp(char c) {
    switch (c) {
        case 'A': return 'T';
        case 'C': return 'G';
        case 'G': return 'C';
        case 'T': return 'A';
        default: return 'N';
    }
}

int n_threads() {
    unsigned h = std::thread::hardware_concurrency();
    return h == 0 ? 1 : static_cast<int>(std::min(h, 64u));
}

template <typename F>
void parallel_chunks(uint64_t n_chunks, F f) {
    int t = std::min<uint64_t>(n_threads(), n_chunks);
    if (t <= 1) {
        for (uint64_t c = 0; c < n_chunks; ++c) f(c);
        return;
    }
    std::vector<std::thread> th;
    for (int i = 0; i < t; ++i)
        th.emplace_back([&, i] {
            for (uint64_t c = i; c < n_chunks; c += t) f(c);
        });
    for (auto& x : th) x.join();
}

inline uint64_t geometric(Xoshiro& rng, double p, int max_len) {
    // number of trials to first success, support {1, 2, ...}, clamped
    uint64_t k = 1;
    while (rng.unit() >= p && k < static_cast<uint64_t>(max_len)) ++k;
    return k;
}

}  // namespace

extern "C" {

void synth_random_genome(uint64_t seed, uint64_t len, char* out) {
    const uint64_t chunk = uint64_t{1} << 26;
    uint64_t n_chunks = (len + chunk - 1) / chunk;
    parallel_chunks(n_chunks, [&](uint64_t c) {
        std::mt19937_64 rng(c == 0 ? seed : splitmix64(seed + c));
        uint64_t b = c * chunk, e = std::min(len, b + chunk);
        for (uint64_t i = b; i < e; ++i) out[i] = kAcgt[rng() % 4];
    });
}

// Repeat-bearing genome (C2/C3 style).  Background = synth_random_genome.
// n_families consensus sequences, length uniform in [min_len, max_len],
// nominal copy count uniform in [min_copies, max_copies], per-family
// divergence uniform in [min_div, max_div] (substitutions; one tenth of that
// rate as 1-base indels).  BASELINE.json's C2 numbers over-specify the repeat
// mass (~16 Gbp of repeats for a 3.1 Gbp genome), so copy counts are scaled by
// one factor so that planted bases total repeat_fraction * len.
// Copies overwrite the background at uniform positions in family order;
// chunks of the genome are patched in parallel, each applying every copy that
// overlaps it in the same global order, so the output is thread-independent.
void synth_repeat_genome(uint64_t seed, uint64_t len, int n_families, int min_len, int max_len,
                         int min_copies, int max_copies, double min_div, double max_div,
                         double repeat_fraction, char* out) {
    synth_random_genome(seed, len, out);
    if (n_families <= 0 || len < static_cast<uint64_t>(max_len) * 2) return;
    struct Family {
        uint64_t len, copies;
        double div;
    };
    Xoshiro fr(splitmix64(seed ^ 0xFA3117ull));
    std::vector<Family> fam(n_families);
    double mass = 0;
    for (auto& f : fam) {
        f.len = min_len + fr() % static_cast<uint64_t>(max_len - min_len + 1);
        f.copies = min_copies + fr() % static_cast<uint64_t>(max_copies - min_copies + 1);
        f.div = min_div + (max_div - min_div) * fr.unit();
        mass += static_cast<double>(f.len) * static_cast<double>(f.copies);
    }
    double scale = repeat_fraction * static_cast<double>(len) / mass;
    struct Copy {
        uint64_t at, fam, idx;
    };
    std::vector<Copy> copies;
    for (uint64_t fi = 0; fi < fam.size(); ++fi) {
        auto& f = fam[fi];
        f.copies = std::max<uint64_t>(
            1, static_cast<uint64_t>(std::llround(static_cast<double>(f.copies) * scale)));
        for (uint64_t c = 0; c < f.copies; ++c)
            copies.push_back({fr() % (len - 2 * f.len), fi, c});
    }
    // consensus per family
    std::vector<std::string> cons(fam.size());
    parallel_chunks(fam.size(), [&](uint64_t fi) {
        Xoshiro r(splitmix64(seed * 31 + fi + 1));
        cons[fi].resize(fam[fi].len);
        for (auto& ch : cons[fi]) ch = kAcgt[r() & 3];
    });
    auto make_copy = [&](const Copy& c, std::string& buf) {
        const Family& f = fam[c.fam];
        Xoshiro r(splitmix64((seed << 20) ^ (c.fam * 0x100000001B3ull) ^ (c.idx + 7)));
        buf.clear();
        const std::string& src = cons[c.fam];
        for (size_t i = 0; i < src.size(); ++i) {
            double u = r.unit();
            if (u < f.div) {
                char b;
                do b = kAcgt[r() & 3]; while (b == src[i]);
                buf += b;
            } else if (u < f.div * 1.1) {
                if (r() & 1) {
                    buf += src[i];
                    buf += kAcgt[r() & 3];
                }
            } else {
                buf += src[i];
            }
        }
    };
    const uint64_t chunk = uint64_t{1} << 24;
    uint64_t n_chunks = (len + chunk - 1) / chunk;
    // bucket copies by the chunks they touch (copy length <= 1.2 * max_len)
    std::vector<std::vector<uint32_t>> touching(n_chunks);
    for (uint32_t i = 0; i < copies.size(); ++i) {
        uint64_t b = copies[i].at, e = std::min(len, b + fam[copies[i].fam].len * 2);
        for (uint64_t c = b / chunk; c <= (e - 1) / chunk; ++c) touching[c].push_back(i);
    }
    parallel_chunks(n_chunks, [&](uint64_t c) {
        std::string buf;
        uint64_t cb = c * chunk, ce = std::min(len, cb + chunk);
        for (uint32_t i : touching[c]) {
            make_copy(copies[i], buf);
            uint64_t b = copies[i].at;
            for (uint64_t j = 0; j < buf.size(); ++j) {
                uint64_t p = b + j;
                if (p >= len) break;
                if (p >= cb && p < ce) out[p] = buf[j];
            }
        }
    });
}

// ASCII -> PackedGenome words (REF src/genome.cpp:39-46 layout).  Returns -1
// on an illegal character.  Chunked over 64-base blocks in parallel.
int synth_pack_genome(const char* seq, uint64_t len, uint64_t* packed, uint64_t* nmask) {
    uint64_t n_blocks = (len + 63) / 64;
    std::vector<int> bad(n_threads() + 1, 0);
    const uint64_t per = 1 << 16;  // blocks per task
    uint64_t tasks = (n_blocks + per - 1) / per;
    std::vector<char> fail(tasks, 0);
    parallel_chunks(tasks, [&](uint64_t t) {
        for (uint64_t blk = t * per; blk < std::min(n_blocks, (t + 1) * per); ++blk) {
            uint64_t w0 = 0, w1 = 0, nm = 0;
            for (int j = 0; j < 64; ++j) {
                uint64_t pos = blk * 64 + j;
                if (pos >= len) break;
                uint64_t code;
                switch (seq[pos]) {
                    case 'A': case 'a': code = 0; break;
                    case 'C': case 'c': code = 1; break;
                    case 'G': case 'g': code = 2; break;
                    case 'T': case 't': code = 3; break;
                    case 'N': case 'n': case 'R': case 'Y': case 'S': case 'W': case 'K':
                    case 'M': case 'B': case 'D': case 'H': case 'V': case 'U':
                    case 'r': case 'y': case 's': case 'w': case 'k': case 'm': case 'b':
                    case 'd': case 'h': case 'v': case 'u':
                        code = 0;
                        nm |= uint64_t{1} << j;
                        break;
                    default: fail[t] = 1; code = 0;
                }
                if (j < 32) w0 |= code << (2 * j);
                else w1 |= code << (2 * (j - 32));
            }
            packed[2 * blk] = w0;
            if (2 * blk + 1 < (len + 31) / 32) packed[2 * blk + 1] = w1;
            nmask[blk] = nm;
        }
    });
    for (char f : fail)
        if (f) return -1;
    return 0;
}

// Fixed-length reads: out holds n_reads * read_len bytes; truth_pos[i] is the
// forward-strand start of the template, truth_dir[i] 0 = forward, 1 = RC.
// Loci whose template would run off the genome or touch N are redrawn.
int synth_reads(const char* genome, uint64_t glen, uint64_t seed, uint64_t n_reads, int read_len,
                double sub_rate, double indel_rate, double geom_p, int max_indel, char* out,
                uint64_t* truth_pos, uint8_t* truth_dir) {
    const uint64_t L = static_cast<uint64_t>(read_len);
    const uint64_t slack = 64 + L / 2 + static_cast<uint64_t>(max_indel) * 4;
    if (glen <= L + slack) return -1;
    const uint64_t per = 4096;
    uint64_t tasks = (n_reads + per - 1) / per;
    parallel_chunks(tasks, [&](uint64_t t) {
        std::string buf;
        buf.reserve(L + static_cast<uint64_t>(max_indel) + 8);
        for (uint64_t i = t * per; i < std::min(n_reads, (t + 1) * per); ++i) {
            Xoshiro rng(splitmix64(seed * 0x2545F4914F6CDD1Dull + i));
            for (int attempt = 0; attempt < 1000; ++attempt) {
                uint64_t start = rng() % (glen - L - slack);
                bool rc = (rng() & 1) != 0;
                buf.clear();
                uint64_t g = start;
                bool ok = true;
                while (buf.size() < L) {
                    if (g >= glen) {
                        ok = false;
                        break;
                    }
                    char base = genome[g];
                    if (base == 'N') {
                        ok = false;
                        break;
                    }
                    double u = rng.unit();
                    if (u < indel_rate) {
                        uint64_t k = geometric(rng, geom_p, max_indel);
                        if (rng() & 1) {
                            for (uint64_t j = 0; j < k; ++j) buf += kAcgt[rng() & 3];
                        } else {
                            g += k;
                        }
                    } else if (u < indel_rate + sub_rate) {
                        char b;
                        do b = kAcgt[rng() & 3]; while (b == base);
                        buf += b;
                        ++g;
                    } else {
                        buf += base;
                        ++g;
                    }
                }
                if (!ok) continue;
                buf.resize(L);
                char* dst = out + i * L;
                if (rc) {
                    for (uint64_t j = 0; j < L; ++j) dst[j] = comp(buf[L - 1 - j]);
                } else {
                    std::memcpy(dst, buf.data(), L);
                }
                if (truth_pos) truth_pos[i] = start;
                if (truth_dir) truth_dir[i] = rc ? 1 : 0;
                break;
            }
        }
    });
    return 0;
}

}  // extern "C"
