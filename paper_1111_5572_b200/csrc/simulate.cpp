// simulate.cpp -- the reference's read simulator behind the C ABI.
//
//   sa_simulator_*   ReadSimulator (REF include/seedaln/simulator.hpp:48-66,
//                    src/simulator.cpp:101-192): same mt19937_64 stream, same
//                    draws in the same order, so reads, names and truths are
//                    identical to the reference's for the same genome/profile
//   sa_run_simulate  run_simulate (REF src/driver.cpp:158-168): FASTA -> FASTQ,
//                    byte-identical to the reference's file
//
// The reference builds every read through four std::strings (extract,
// mutated, observed, the reverse complement) and compares each draw as a
// double.  Here one read is produced in reusable buffers, the genome window is
// decoded from the packed words 32 bases at a time, and each rate test is the
// exact integer form of the reference's double compare:
//   (r >> 11) * 2^-53 < p   <=>   (r >> 11) < ceil(p * 2^53)
// (both sides are exact: r >> 11 < 2^53 and scaling by 2^53 is exact).
// The draws are one sequential stream (REF simulator.cpp:104), so generation
// is one thread; run_sa_simulate formats FASTQ records on the other host
// cores while the next batch is generated.
#include <immintrin.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <future>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "host_common.h"

using sab::fail_thread;

namespace {

constexpr char kAcgt[4] = {'A', 'C', 'G', 'T'};  // REF simulator.cpp:11
constexpr int kMaxPlacementAttempts = 10000;      // REF simulator.cpp:12

// integer threshold T with  unit_real(r) < p  <=>  (r >> 11) < T  (REF simulator.cpp:26-28)
uint64_t rate_threshold(double p) {
    if (!(p > 0.0)) return 0;
    const double y = std::ceil(std::ldexp(p, 53));
    return y >= 18446744073709551615.0 ? ~uint64_t{0} : static_cast<uint64_t>(y);
}

// std::mt19937_64 (the reference's engine, REF simulator.hpp:62): same
// seeding, twist and tempering, but a whole state's 312 outputs are made at
// once (AVX2 when the host has it), together with two bitmaps marking the
// draws below the two rate thresholds the read loops scan for, so a run of
// draws with no event is found with one count-trailing-zeros.
class Mt64 {
  public:
    static constexpr int kN = 312, kM = 156, kW = (kN + 63) / 64;
    void seed(uint64_t s, uint64_t t0, uint64_t t1) {
        mt_[0] = s;
        for (int i = 1; i < kN; ++i) mt_[i] = 6364136223846793005ull * (mt_[i - 1] ^ (mt_[i - 1] >> 62)) + i;
        t_[0] = t0;
        t_[1] = t1;
        pos_ = kN;
        fill_ = __builtin_cpu_supports("avx2") ? &Mt64::refill_avx2 : &Mt64::refill_scalar;
    }
    uint64_t operator()() {
        if (pos_ == kN) (this->*fill_)();
        return out_[pos_++];
    }
    int avail() {
        if (pos_ == kN) (this->*fill_)();
        return kN - pos_;
    }
    // leading draws among the next n (n <= avail()) that are not below threshold `which`
    int quiet(int which, int n) const {
        const uint64_t* ev = ev_[which];
        int p = pos_;
        const int end = pos_ + n;
        while (p < end) {
            const uint64_t m = ev[p >> 6] >> (p & 63);
            if (m) return std::min(end, p + __builtin_ctzll(m)) - pos_;
            p = (p | 63) + 1;
        }
        return n;
    }
    void skip(int n) { pos_ += n; }

  private:
    static uint64_t twist(uint64_t a, uint64_t b, uint64_t c) {
        const uint64_t x = (a & 0xFFFFFFFF80000000ull) | (b & 0x7FFFFFFFull);
        return c ^ (x >> 1) ^ ((0 - (x & 1)) & 0xB5026F5AA96619E9ull);
    }
    static uint64_t temper(uint64_t y) {
        y ^= (y >> 29) & 0x5555555555555555ull;
        y ^= (y << 17) & 0x71D67FFFEDA60000ull;
        y ^= (y << 37) & 0xFFF7EEE000000000ull;
        return y ^ (y >> 43);
    }
    void refill_scalar() {
        int i = 0;
        for (; i < kN - kM; ++i) mt_[i] = twist(mt_[i], mt_[i + 1], mt_[i + kM]);
        for (; i < kN - 1; ++i) mt_[i] = twist(mt_[i], mt_[i + 1], mt_[i + kM - kN]);
        mt_[kN - 1] = twist(mt_[kN - 1], mt_[0], mt_[kM - 1]);
        for (int w = 0; w < kW; ++w) ev_[0][w] = ev_[1][w] = 0;
        for (int k = 0; k < kN; ++k) {
            out_[k] = temper(mt_[k]);
            ev_[0][k >> 6] |= static_cast<uint64_t>((out_[k] >> 11) < t_[0]) << (k & 63);
            ev_[1][k >> 6] |= static_cast<uint64_t>((out_[k] >> 11) < t_[1]) << (k & 63);
        }
        pos_ = 0;
    }
    __attribute__((target("avx2"))) static __m256i twist4(__m256i a, __m256i b, __m256i c) {
        const __m256i x = _mm256_or_si256(_mm256_and_si256(a, _mm256_set1_epi64x(0xFFFFFFFF80000000ull)),
                                          _mm256_and_si256(b, _mm256_set1_epi64x(0x7FFFFFFFull)));
        const __m256i odd = _mm256_sub_epi64(_mm256_setzero_si256(), _mm256_and_si256(x, _mm256_set1_epi64x(1)));
        return _mm256_xor_si256(_mm256_xor_si256(c, _mm256_srli_epi64(x, 1)),
                                _mm256_and_si256(odd, _mm256_set1_epi64x(0xB5026F5AA96619E9ull)));
    }
    __attribute__((target("avx2"))) void refill_avx2() {
#define ld(q) _mm256_loadu_si256(reinterpret_cast<const __m256i*>(q))
        int i = 0;
        for (; i < kN - kM; i += 4)  // 156 = 39 x 4; mt[i+1..i+4] are still the old values
            _mm256_storeu_si256(reinterpret_cast<__m256i*>(mt_ + i), twist4(ld(mt_ + i), ld(mt_ + i + 1), ld(mt_ + i + kM)));
        for (; i + 4 < kN; i += 4)   // mt[i-156..] were updated by the first loop
            _mm256_storeu_si256(reinterpret_cast<__m256i*>(mt_ + i),
                                twist4(ld(mt_ + i), ld(mt_ + i + 1), ld(mt_ + i + kM - kN)));
        for (; i < kN - 1; ++i) mt_[i] = twist(mt_[i], mt_[i + 1], mt_[i + kM - kN]);
        mt_[kN - 1] = twist(mt_[kN - 1], mt_[0], mt_[kM - 1]);
        const __m256i T0 = _mm256_set1_epi64x(static_cast<long long>(t_[0]));
        const __m256i T1 = _mm256_set1_epi64x(static_cast<long long>(t_[1]));
        for (int w = 0; w < kW; ++w) ev_[0][w] = ev_[1][w] = 0;
        for (int k = 0; k < kN; k += 4) {  // 312 = 78 x 4
            __m256i y = ld(mt_ + k);
            y = _mm256_xor_si256(y, _mm256_and_si256(_mm256_srli_epi64(y, 29), _mm256_set1_epi64x(0x5555555555555555ull)));
            y = _mm256_xor_si256(y, _mm256_and_si256(_mm256_slli_epi64(y, 17), _mm256_set1_epi64x(0x71D67FFFEDA60000ull)));
            y = _mm256_xor_si256(y, _mm256_and_si256(_mm256_slli_epi64(y, 37), _mm256_set1_epi64x(0xFFF7EEE000000000ull)));
            y = _mm256_xor_si256(y, _mm256_srli_epi64(y, 43));
            _mm256_storeu_si256(reinterpret_cast<__m256i*>(out_ + k), y);
            const __m256i x = _mm256_srli_epi64(y, 11);  // < 2^53 and thresholds <= 2^53: signed compare is exact
            const uint64_t m0 = static_cast<uint64_t>(_mm256_movemask_pd(_mm256_castsi256_pd(_mm256_cmpgt_epi64(T0, x))));
            const uint64_t m1 = static_cast<uint64_t>(_mm256_movemask_pd(_mm256_castsi256_pd(_mm256_cmpgt_epi64(T1, x))));
            ev_[0][k >> 6] |= m0 << (k & 63);
            ev_[1][k >> 6] |= m1 << (k & 63);
        }
#undef ld
        pos_ = 0;
    }
    uint64_t mt_[kN];
    uint64_t out_[kN];
    uint64_t ev_[2][kW];
    uint64_t t_[2] = {0, 0};
    int pos_ = kN;
    void (Mt64::*fill_)() = &Mt64::refill_scalar;
};

struct RateError {
    std::string msg;
};

// SimProfile::validate (REF simulator.cpp:31-41)
void validate(const sa_sim_profile& p) {
    if (p.read_length < 1) throw RateError{"read length must be >= 1"};
    auto rate = [](double r, const char* what) {
        if (!(r >= 0.0 && r <= 1.0)) throw RateError{std::string(what) + " must be in [0, 1]"};
    };
    rate(p.snp_rate, "snp rate");
    rate(p.indel_mutation_rate, "indel mutation rate");
    rate(p.seq_error_rate, "sequencing error rate");
    rate(p.indel_error_fraction, "indel error fraction");
}

}  // namespace

struct sa_simulator {
    const sa_genome* g = nullptr;
    sa_sim_profile p{};
    Mt64 rng;
    uint64_t serial = 0, placeable = 0;
    uint64_t t_snp = 0, t_mut = 0, t_err = 0, t_ierr = 0;
    // placeable contigs: (global start, span, cumulative span before, contig index)
    struct Span {
        uint64_t start, span, before, index;
    };
    std::vector<Span> spans;
    std::vector<char> extract, mutated, observed;
    const char* ex = nullptr;  // the decoded window: ex[0, ne)
    size_t ne = 0;

    char base() { return kAcgt[rng() & 3]; }  // REF simulator.cpp:14-16
    char other(char c) {                      // REF simulator.cpp:18-24
        char b;
        do {
            b = base();
        } while (b == c);
        return b;
    }
    bool below(uint64_t t) { return (rng() >> 11) < t; }

    // REF simulator.cpp:101-115: u = rng() % placeable, walk the contigs
    // skipping short ones (a binary search over the cumulative spans).
    const Span& pick(uint64_t& offset) {
        const uint64_t u = rng() % placeable;
        auto it = std::upper_bound(spans.begin(), spans.end(), u,
                                   [](uint64_t v, const Span& s) { return v < s.before; });
        const Span& s = *(it - 1);
        offset = u - s.before;
        return s;
    }

    // PackedGenome::substring (REF genome.cpp:114-123) into `extract`:
    // 4 bases per packed byte through a table, N bits applied after.
    void decode(uint64_t pos, uint64_t len) {
        static const struct Lut {
            uint32_t v[256];
            Lut() {
                for (int b = 0; b < 256; ++b) {
                    uint32_t w = 0;
                    for (int j = 0; j < 4; ++j) w |= static_cast<uint32_t>(static_cast<uint8_t>(kAcgt[(b >> (2 * j)) & 3])) << (8 * j);
                    v[b] = w;
                }
            }
        } lut;
        const uint64_t n = std::min(len, g->length - pos);
        const uint64_t a = pos & ~uint64_t{3}, e = (pos + n + 3) & ~uint64_t{3};
        if (extract.size() < e - a) extract.resize(e - a);
        const uint8_t* bytes = reinterpret_cast<const uint8_t*>(g->packed.data());
        for (uint64_t q = a, o = 0; q < e; q += 4, o += 4) {
            const uint64_t byte = q >> 2;  // the last byte may lie past the genome end in the final word
            std::memcpy(extract.data() + o, &lut.v[byte < 8 * g->packed.size() ? bytes[byte] : 0], 4);
        }
        for (uint64_t q = pos & ~uint64_t{63}; q < pos + n; q += 64) {  // N bits
            uint64_t m = g->nmask[q >> 6];
            while (m) {
                const uint64_t at = q + __builtin_ctzll(m);
                m &= m - 1;
                if (at >= pos && at < pos + n) extract[at - a] = 'N';
            }
        }
        ex = extract.data() + (pos - a);
        ne = n;
    }

    void germline_event(size_t& i, uint64_t x) {  // REF simulator.cpp:148-156, one non-N base
        const char b = ex[i];
        if (x < t_snp) {
            mutated.push_back(other(b));
            ++i;
        } else {
            const size_t k = 1 + rng() % 3;
            if ((rng() & 1) != 0) {
                mutated.push_back(b);
                for (size_t j = 0; j < k; ++j) mutated.push_back(base());
                ++i;
            } else {
                i += k;  // deletion
            }
        }
    }
    void seq_error(char b) {  // REF simulator.cpp:170-180, after r < seq_error_rate
        if (below(t_ierr)) {
            if ((rng() & 1) != 0) {
                observed.push_back(b);
                observed.push_back(base());
            }  // else: single-base deletion
        } else {
            observed.push_back(b == 'N' ? base() : other(b));
        }
    }

    // germline mutations (REF simulator.cpp:136-159) then sequencing errors
    // (REF :162-181).  no_n: the window holds no N, so every base draws once
    // and runs of draws without an event are copied in bulk.
    void mutate(uint64_t len, bool no_n) {
        mutated.clear();
        if (no_n) {
            for (size_t i = 0; i < ne;) {
                const int n = static_cast<int>(std::min<size_t>(rng.avail(), ne - i));
                const int j = rng.quiet(0, n);
                mutated.insert(mutated.end(), ex + i, ex + i + j);
                rng.skip(j);
                i += j;
                if (j < n) germline_event(i, rng() >> 11);
            }
        } else {
            for (size_t i = 0; i < ne;) {
                if (ex[i] == 'N') {
                    mutated.push_back('N');
                    ++i;
                    continue;
                }
                const uint64_t x = rng() >> 11;
                if (x < t_mut) {
                    germline_event(i, x);
                } else {
                    mutated.push_back(ex[i]);
                    ++i;
                }
            }
        }
        observed.clear();
        const size_t nm = mutated.size(), cap = len + 8;
        for (size_t i = 0; i < nm && observed.size() < cap;) {
            // bases before the cap, each one draw; a quiet run is copied
            const int n = static_cast<int>(std::min<size_t>({static_cast<size_t>(rng.avail()), nm - i,
                                                             cap - observed.size()}));
            const int j = rng.quiet(1, n);
            observed.insert(observed.end(), mutated.begin() + i, mutated.begin() + i + j);
            rng.skip(j);
            i += j;
            if (j < n) {
                rng.skip(1);  // the draw that was below seq_error_rate
                seq_error(mutated[i++]);
            }
        }
    }

    // ReadSimulator::next (REF simulator.cpp:117-192): bases (read_length
    // chars) and the truth.
    bool next(char* out, sa_sim_truth& truth) {
        const uint64_t len = p.read_length;
        const uint64_t slack = 64 + len / 4;  // REF :128
        for (int attempt = 0; attempt < kMaxPlacementAttempts; ++attempt) {
            uint64_t offset = 0;
            const Span& sp = pick(offset);
            const uint64_t global = sp.start + offset;
            const bool reverse = (rng() & 1) != 0;  // REF :124

            decode(global, len + slack);
            if (ne < len) continue;
            if (std::memchr(ex, 'N', len) != nullptr) continue;  // REF :131-133

            mutate(len, std::memchr(ex, 'N', ne) == nullptr);
            if (observed.size() < len) continue;  // REF :183
            if (std::memchr(observed.data(), 'N', len) != nullptr) continue;  // REF :185

            truth.contig = sp.index;
            truth.position = offset;
            truth.direction = reverse ? SA_REVERSE_COMPLEMENT : SA_FORWARD;
            truth.serial = serial++;
            if (!reverse) {
                std::memcpy(out, observed.data(), len);
            } else {  // reverse_complement (REF genome.cpp:182-200); no N left here
                static const struct Comp {
                    char v[256];
                    Comp() {
                        for (int c = 0; c < 256; ++c) v[c] = 'A';
                        v['A'] = 'T';
                        v['C'] = 'G';
                        v['G'] = 'C';
                    }
                } comp;
                const char* o = observed.data() + len - 1;
                for (uint64_t i = 0; i < len; ++i) out[i] = comp.v[static_cast<uint8_t>(o[-static_cast<int64_t>(i)])];
            }
            return true;
        }
        return false;
    }
};

namespace {

// encode_truth + to_fastq (REF simulator.cpp:43-48, 194-206) for reads
// [r0, r1) of a batch; returns the bytes written (out == nullptr: size only).
uint64_t format_fastq(const sa_genome& g, uint64_t len, const char* bases, const sa_sim_truth* truth,
                      uint64_t r0, uint64_t r1, char* out) {
    uint64_t n = 0;
    char num[2][24];
    for (uint64_t r = r0; r < r1; ++r) {
        const sa_sim_truth& t = truth[r];
        const std::string& cname = g.contigs[t.contig].name;
        const int l1 = snprintf(num[0], sizeof num[0], "%llu", static_cast<unsigned long long>(t.position + 1));
        const int l2 = snprintf(num[1], sizeof num[1], "%llu", static_cast<unsigned long long>(t.serial));
        const uint64_t rec = 1 + cname.size() + 1 + l1 + 3 + l2 + 1 + len + 3 + len + 1;
        if (out) {
            char* o = out + n;
            *o++ = '@';
            std::memcpy(o, cname.data(), cname.size());
            o += cname.size();
            *o++ = '_';
            std::memcpy(o, num[0], l1);
            o += l1;
            *o++ = '_';
            *o++ = t.direction == SA_FORWARD ? 'F' : 'R';
            *o++ = '_';
            std::memcpy(o, num[1], l2);
            o += l2;
            *o++ = '\n';
            std::memcpy(o, bases + r * len, len);
            o += len;
            *o++ = '\n';
            *o++ = '+';
            *o++ = '\n';
            std::memset(o, 'I', len);
            o += len;
            *o++ = '\n';
        }
        n += rec;
    }
    return n;
}

}  // namespace

extern "C" {

void sa_default_sim_profile(sa_sim_profile* out) {  // SimProfile{} (REF simulator.hpp:17-24)
    out->read_length = 100;
    out->snp_rate = 0.0009;
    out->indel_mutation_rate = 0.0001;
    out->seq_error_rate = 0.02;
    out->indel_error_fraction = 0.0;
    out->rng_seed = 1;
}

int sa_simulator_create(const sa_genome* g, const sa_sim_profile* p, sa_simulator** out) {
    if (!g || !p || !out) return fail_thread(SA_EINVAL, "null argument");
    *out = nullptr;
    try {
        validate(*p);
    } catch (const RateError& e) {
        return fail_thread(SA_EINVAL, e.msg);
    }
    auto* s = new sa_simulator;
    s->g = g;
    s->p = *p;
    for (size_t i = 0; i < g->contigs.size(); ++i) {  // REF simulator.cpp:92-94
        const auto& c = g->contigs[i];
        if (c.length >= p->read_length) {
            const uint64_t span = c.length - p->read_length + 1;
            s->spans.push_back({c.start, span, s->placeable, i});
            s->placeable += span;
        }
    }
    if (s->placeable == 0) {  // REF simulator.cpp:95-98
        delete s;
        return fail_thread(SA_EINVAL, "no contig is long enough for the requested read length");
    }
    // REF :150 compares r < snp and r < snp + indel (the sum rounded as a double)
    s->t_snp = rate_threshold(p->snp_rate);
    s->t_mut = rate_threshold(p->snp_rate + p->indel_mutation_rate);
    s->t_err = rate_threshold(p->seq_error_rate);
    s->t_ierr = rate_threshold(p->indel_error_fraction);
    s->rng.seed(p->rng_seed, s->t_mut, s->t_err);  // bitmaps for the two bulk-scanned tests
    *out = s;
    return SA_OK;
}

void sa_simulator_destroy(sa_simulator* s) { delete s; }

int sa_simulator_next(sa_simulator* s, uint64_t count, char* bases, sa_sim_truth* truth) {
    if (!s || (count && (!bases || !truth))) return fail_thread(SA_EINVAL, "null argument");
    const uint64_t len = s->p.read_length;
    for (uint64_t r = 0; r < count; ++r)
        if (!s->next(bases + r * len, truth[r]))  // REF simulator.cpp:190-191
            return fail_thread(SA_ERUNTIME, "failed to place a read; genome may be mostly N");
    return SA_OK;
}

int sa_run_simulate(const char* fasta_path, const char* output_path, uint64_t count, const sa_sim_profile* p,
                    uint32_t threads) {
    if (!fasta_path || !output_path || !p) return fail_thread(SA_EINVAL, "null argument");
    if (count < 1) return fail_thread(SA_EINVAL, "read count must be >= 1");  // REF driver.cpp:159
    sa_genome* g = nullptr;
    if (int rc = sa_genome_from_fasta(fasta_path, &g)) return rc;  // REF driver.cpp:160-161
    std::unique_ptr<sa_genome, void (*)(sa_genome*)> gh(g, sa_genome_free);
    sa_simulator* sim = nullptr;
    if (int rc = sa_simulator_create(g, p, &sim)) return rc;  // REF driver.cpp:162
    std::unique_ptr<sa_simulator, void (*)(sa_simulator*)> sh(sim, sa_simulator_destroy);
    FILE* f = fopen(output_path, "wb");  // REF driver.cpp:163 open_output
    if (!f) return fail_thread(SA_EIO, std::string("cannot open ") + output_path + " for writing");
    std::unique_ptr<FILE, int (*)(FILE*)> fh(f, fclose);

    const uint64_t len = p->read_length;
    const uint64_t batch = std::max<uint64_t>(1, std::min<uint64_t>(count, (64ull << 20) / (len + 64)));
    unsigned nt = threads ? threads : std::max(1u, std::thread::hardware_concurrency());
    struct Batch {
        std::vector<char> bases;
        std::vector<sa_sim_truth> truth;
        uint64_t n = 0;
        int rc = SA_OK;
    };
    Batch buf[2];
    auto generate = [&](Batch& b, uint64_t n) {
        b.n = n;
        b.bases.resize(n * len);
        b.truth.resize(n);
        b.rc = SA_OK;
        for (uint64_t r = 0; r < n; ++r)
            if (!sim->next(b.bases.data() + r * len, b.truth[r])) {  // REF simulator.cpp:190-191
                b.n = r;
                b.rc = fail_thread(SA_ERUNTIME, "failed to place a read; genome may be mostly N");
                break;
            }
    };
    std::vector<char> text;
    uint64_t done = 0;
    generate(buf[0], std::min(batch, count));
    for (int cur = 0;; cur ^= 1) {
        Batch& b = buf[cur];
        done += b.n;
        std::future<void> nxt;
        if (done < count && b.rc == SA_OK)  // the next batch is generated while this one is formatted and written
            nxt = std::async(std::launch::async, generate, std::ref(buf[cur ^ 1]), std::min(batch, count - done));
        const unsigned parts = std::max(1u, std::min<unsigned>(nt, static_cast<unsigned>((b.n + 1023) / 1024)));
        std::vector<uint64_t> off(parts + 1, 0);
        auto range = [&](unsigned k, uint64_t& r0, uint64_t& r1) {
            r0 = b.n * k / parts;
            r1 = b.n * (k + 1) / parts;
        };
        {
            std::vector<std::thread> th;
            for (unsigned k = 0; k < parts; ++k)
                th.emplace_back([&, k] {
                    uint64_t r0, r1;
                    range(k, r0, r1);
                    off[k + 1] = format_fastq(*g, len, b.bases.data(), b.truth.data(), r0, r1, nullptr);
                });
            for (auto& t : th) t.join();
        }
        for (unsigned k = 0; k < parts; ++k) off[k + 1] += off[k];
        text.resize(off[parts]);
        {
            std::vector<std::thread> th;
            for (unsigned k = 0; k < parts; ++k)
                th.emplace_back([&, k] {
                    uint64_t r0, r1;
                    range(k, r0, r1);
                    format_fastq(*g, len, b.bases.data(), b.truth.data(), r0, r1, text.data() + off[k]);
                });
            for (auto& t : th) t.join();
        }
        const bool wrote = fwrite(text.data(), 1, text.size(), f) == text.size();
        if (nxt.valid()) nxt.get();
        if (!wrote) return fail_thread(SA_EIO, std::string("failed writing ") + output_path);
        if (b.rc) {  // the reads before the failure are in the file, as the reference's stream has them
            fflush(f);
            return b.rc;
        }
        if (done >= count) break;
    }
    if (fflush(f) != 0) return fail_thread(SA_EIO, std::string("failed writing ") + output_path);
    return SA_OK;
}

}  // extern "C"
