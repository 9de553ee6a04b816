// run_align.cpp -- FASTQ -> SAM through the GPU batcher.
//
// Follows run_align (REF src/driver.cpp:47-156) and the pieces it calls:
//   FASTQ records and record-start resync  REF src/fastq.cpp:11-99
//   ChunkScheduler / next_chunk           REF src/scheduler.cpp:8-31
//   sam_header / make_sam_record / format REF src/sam.cpp:11-87
//   decode_truth                          REF src/simulator.cpp:50-78
//   score_result / EvalReport             REF src/eval.cpp:12-120
// Workers take byte-range chunks from the same scheduler; a chunk owns the
// records whose first byte lies inside it.  Each worker parses its chunk,
// aligns all of the chunk's reads in one sa_align_batch call (the GPU; calls
// are serialised on the context, parsing and formatting run in parallel),
// scores and formats them, and hands the text to the ordered writer.  With
// stable_order the output is byte-identical to the reference's; without it,
// chunks are written as they complete.
#include <algorithm>
#include <atomic>
#include <cerrno>
#include <charconv>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fcntl.h>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <sys/stat.h>
#include <thread>
#include <unistd.h>
#include <vector>

#include "host_common.h"

using sab::fail_thread;

namespace {

struct Error {
    int code;
    std::string msg;
};

// ---------------------------------------------------------------- input file

class InFile {  // positional reads; lines as the reference's std::getline sees them
public:
    explicit InFile(const std::string& path) : fd_(open(path.c_str(), O_RDONLY)) {}
    ~InFile() {
        if (fd_ >= 0) close(fd_);
    }
    bool ok() const { return fd_ >= 0; }
    int fd() const { return fd_; }

private:
    int fd_;
};

// Sequential line reader from a byte offset (getline semantics: the newline is
// consumed and not returned; the last line may lack one).
class LineReader {
public:
    LineReader(int fd, uint64_t at) : fd_(fd), pos_(at) {}
    // false at end of input; `had_newline` tells whether '\n' ended the line
    bool line(std::string& out, bool& had_newline) {
        out.clear();
        for (;;) {
            if (i_ == n_) {
                if (!fill()) {
                    had_newline = false;
                    return !out.empty();
                }
            }
            const char* s = buf_.data() + i_;
            const void* nl = std::memchr(s, '\n', n_ - i_);
            if (nl) {
                const size_t k = static_cast<const char*>(nl) - s;
                out.append(s, k);
                i_ += k + 1;
                had_newline = true;
                return true;
            }
            out.append(s, n_ - i_);
            i_ = n_;
        }
    }
    bool at_eof() {  // peek() == EOF
        if (i_ < n_) return false;
        return !fill();
    }

private:
    bool fill() {
        if (buf_.empty()) buf_.resize(1 << 20);
        ssize_t r;
        do {
            r = pread(fd_, buf_.data(), buf_.size(), static_cast<off_t>(pos_));
        } while (r < 0 && errno == EINTR);
        if (r <= 0) {
            i_ = n_ = 0;
            return false;
        }
        pos_ += static_cast<uint64_t>(r);
        i_ = 0;
        n_ = static_cast<size_t>(r);
        return true;
    }
    int fd_;
    uint64_t pos_;
    std::vector<char> buf_;
    size_t i_ = 0, n_ = 0;
};

// REF src/fastq.cpp:66-99 find_fastq_record_start
uint64_t find_record_start(int fd, uint64_t from, uint64_t file_size) {
    if (from >= file_size) return file_size;
    uint64_t pos = from;
    std::string l0, l1, l2;
    bool nl;
    if (from != 0) {
        char c = 0;
        if (pread(fd, &c, 1, static_cast<off_t>(from - 1)) != 1) return file_size;
        if (c != '\n') {
            LineReader r(fd, from);
            if (!r.line(l0, nl)) return file_size;
            pos = from + l0.size() + 1;
        }
    }
    while (pos < file_size) {
        LineReader r(fd, pos);
        if (!r.line(l0, nl)) return file_size;
        const uint64_t next = pos + l0.size() + 1;
        if (!l0.empty() && l0[0] == '@') {
            if (!r.line(l1, nl)) return file_size;
            if (r.line(l2, nl) && !l2.empty() && l2[0] == '+') return pos;
        }
        pos = next;
    }
    return file_size;
}

struct Reads {  // one chunk's records, packed
    std::vector<char> names, bases, quals;
    std::vector<uint64_t> name_off{0}, base_off{0};  // quals share base_off
};

// REF src/fastq.cpp:11-64 FastqReader over [start, ...) while offset < end.
void parse_chunk(int fd, uint64_t start, uint64_t end, Reads& out) {
    LineReader r(fd, start);
    uint64_t offset = start;
    std::string name_line, bases, plus, quals;
    auto get_line = [&](std::string& l) -> bool {
        bool nl;
        if (!r.line(l, nl)) return false;
        offset += l.size() + (nl ? 1 : 0);
        if (!l.empty() && l.back() == '\r') l.pop_back();
        return true;
    };
    while (offset < end) {
        const uint64_t record_start = offset;
        if (!get_line(name_line)) return;
        if (name_line.empty() && r.at_eof()) return;
        auto at = [&] { return std::to_string(record_start); };  // error messages only
        if (name_line.empty() || name_line[0] != '@')
            throw Error{SA_EPARSE, "FASTQ record at byte " + at() + " does not start with '@'"};
        size_t nend = name_line.find_first_of(" \t");
        if (nend == std::string::npos) nend = name_line.size();
        if (nend <= 1) throw Error{SA_EPARSE, "FASTQ record at byte " + at() + " has an empty name"};
        if (!get_line(bases) || !get_line(plus) || !get_line(quals))
            throw Error{SA_EPARSE, "truncated FASTQ record at byte " + at()};
        if (plus.empty() || plus[0] != '+')
            throw Error{SA_EPARSE, "FASTQ record at byte " + at() + " lacks its '+' separator"};
        if (bases.size() != quals.size())
            throw Error{SA_EPARSE, "FASTQ record at byte " + at() + ": base and quality lengths differ"};
        static const struct Norm {  // char_to_code as a table: 'A'..'N' or 0 (illegal)
            char v[256];
            Norm() {
                for (int c = 0; c < 256; ++c) {
                    const int code = sab::char_to_code(static_cast<char>(c));
                    v[c] = code < 0 ? 0 : "ACGTN"[code];
                }
            }
        } norm;
        for (char& ch : bases) {  // uppercase, IUPAC -> N (REF fastq.cpp:52-60)
            const char n = norm.v[static_cast<unsigned char>(ch)];
            if (n == 0) throw Error{SA_EPARSE, "FASTQ record at byte " + at() + ": illegal base character"};
            ch = n;
        }
        out.names.insert(out.names.end(), name_line.begin() + 1, name_line.begin() + static_cast<long>(nend));
        out.name_off.push_back(out.names.size());
        out.bases.insert(out.bases.end(), bases.begin(), bases.end());
        out.quals.insert(out.quals.end(), quals.begin(), quals.end());
        out.base_off.push_back(out.bases.size());
    }
}

// ---------------------------------------------------------------- truth, SAM, report

struct Truth {  // REF include/seedaln/simulator.hpp:30-36
    std::string_view contig;
    uint64_t position;
    int direction;
};

// REF src/simulator.cpp:50-78 decode_truth: "contig_pos1_F|R_serial"
std::optional<Truth> decode_truth(std::string_view name) {
    const size_t u3 = name.rfind('_');
    if (u3 == std::string_view::npos || u3 == 0) return std::nullopt;
    const size_t u2 = name.rfind('_', u3 - 1);
    if (u2 == std::string_view::npos || u2 == 0) return std::nullopt;
    const size_t u1 = name.rfind('_', u2 - 1);
    if (u1 == std::string_view::npos || u1 == 0) return std::nullopt;
    const std::string_view pos_s = name.substr(u1 + 1, u2 - u1 - 1);
    const std::string_view dir_s = name.substr(u2 + 1, u3 - u2 - 1);
    const std::string_view ser_s = name.substr(u3 + 1);
    if (dir_s != "F" && dir_s != "R") return std::nullopt;
    uint64_t pos1 = 0, serial = 0;
    auto [pp, pe] = std::from_chars(pos_s.data(), pos_s.data() + pos_s.size(), pos1);
    if (pe != std::errc() || pp != pos_s.data() + pos_s.size() || pos1 == 0) return std::nullopt;
    auto [sp, se] = std::from_chars(ser_s.data(), ser_s.data() + ser_s.size(), serial);
    if (se != std::errc() || sp != ser_s.data() + ser_s.size()) return std::nullopt;
    return Truth{name.substr(0, u1), pos1 - 1, dir_s == "F" ? SA_FORWARD : SA_REVERSE_COMPLEMENT};
}

enum Score { kCorrect, kWrong, kNotConfident };

struct Report {  // REF include/seedaln/eval.hpp:24-46
    uint64_t total = 0, single = 0, multiple = 0, notfound = 0, correct = 0, wrong = 0, no_truth = 0;
    void add(int kind, std::optional<Score> score) {  // REF src/eval.cpp:35-48
        total++;
        if (kind == SA_SINGLE_HIT) single++;
        else if (kind == SA_MULTIPLE_HITS) multiple++;
        else notfound++;
        if (!score) {
            if (kind == SA_SINGLE_HIT) no_truth++;
            return;
        }
        if (*score == kCorrect) correct++;
        if (*score == kWrong) wrong++;
    }
    void merge(const Report& o) {
        total += o.total;
        single += o.single;
        multiple += o.multiple;
        notfound += o.notfound;
        correct += o.correct;
        wrong += o.wrong;
        no_truth += o.no_truth;
    }
};

void put_u64(std::string& s, uint64_t v) {
    char b[24];
    auto [p, e] = std::to_chars(b, b + sizeof b, v);
    s.append(b, p);
}

void put_i64(std::string& s, int64_t v) {
    char b[24];
    auto [p, e] = std::to_chars(b, b + sizeof b, v);
    s.append(b, p);
}

char complement(char c) {
    switch (c) {
        case 'A': return 'T';
        case 'C': return 'G';
        case 'G': return 'C';
        case 'T': return 'A';
        default: return 'N';
    }
}

// make_sam_record + format_sam_record (REF src/sam.cpp:22-87)
void format_record(std::string& line, const sa_genome& g, const sa_result& res, std::string_view name,
                   std::string_view bases, std::string_view quals) {
    line.append(name);
    const bool mapped = res.has_position != 0;
    const bool rc = mapped && res.direction == SA_REVERSE_COMPLEMENT;
    size_t ci = 0;
    if (mapped) ci = g.contig_of(res.position);
    line += '\t';
    put_u64(line, mapped ? (rc ? 16u : 0u) : 4u);
    line += '\t';
    if (mapped) line += g.contigs[ci].name;
    else line += '*';
    line += '\t';
    put_u64(line, mapped ? res.position - g.contigs[ci].start + 1 : 0);
    line += '\t';
    put_i64(line, mapped && res.kind == SA_SINGLE_HIT ? std::min(60, 10 * res.gap) : 0);
    line += '\t';
    if (mapped) {
        put_u64(line, bases.size());
        line += 'M';
    } else {
        line += '*';
    }
    line += "\t*\t0\t0\t";
    if (bases.empty()) {
        line += '*';
    } else if (rc) {
        const size_t o = line.size(), n = bases.size();
        line.resize(o + n);
        char* d = &line[o];
        for (size_t i = 0; i < n; ++i) d[i] = complement(bases[n - 1 - i]);
    } else {
        line.append(bases);
    }
    line += '\t';
    if (quals.empty()) {
        line += '*';
    } else if (rc) {
        const size_t o = line.size(), n = quals.size();
        line.resize(o + n);
        char* d = &line[o];
        for (size_t i = 0; i < n; ++i) d[i] = quals[n - 1 - i];
    } else {
        line.append(quals);
    }
    if (mapped) {
        line += "\tNM:i:";
        put_i64(line, res.distance);
    }
    line += "\tXR:A:";
    line += res.kind == SA_SINGLE_HIT ? 'S' : (res.kind == SA_MULTIPLE_HITS ? 'M' : 'N');
    line += '\n';
}

std::string sam_header(const sa_genome& g, const char* command_line) {  // REF src/sam.cpp:11-20
    std::string h = "@HD\tVN:1.6\tSO:unknown\n";
    for (const auto& c : g.contigs) {
        h += "@SQ\tSN:" + c.name + "\tLN:";
        put_u64(h, c.length);
        h += '\n';
    }
    h += "@PG\tID:seedaln\tPN:seedaln\tCL:";
    h += command_line ? command_line : "seedaln align";
    h += '\n';
    return h;
}

std::string fixed4(double v) {
    char b[64];
    snprintf(b, sizeof b, "%.4f", v);
    return b;
}

// EvalReport::to_text (REF src/eval.cpp:75-120)
std::string report_text(const sa_eval_report& r) {
    const sa_stats& s = r.stats;
    std::string o;
    auto kv = [&o](const char* k, const std::string& v) {
        o += k;
        o += '=';
        o += v;
        o += '\n';
    };
    auto u = [](uint64_t v) { return std::to_string(v); };
    kv("total", u(r.total));
    kv("single", u(r.single));
    kv("multiple", u(r.multiple));
    kv("notfound", u(r.notfound));
    kv("aligned_pct", fixed4(r.total == 0 ? 0.0 : 100.0 * static_cast<double>(r.single) / static_cast<double>(r.total)));
    if (r.correct + r.wrong > 0)
        kv("error_pct", fixed4(100.0 * static_cast<double>(r.wrong) / static_cast<double>(r.correct + r.wrong)));
    else
        kv("error_pct", "na");
    kv("correct", u(r.correct));
    kv("wrong", u(r.wrong));
    kv("no_truth", u(r.no_truth));
    kv("elapsed_sec", fixed4(r.elapsed_seconds));
    kv("reads_per_sec", fixed4(r.elapsed_seconds > 0 ? static_cast<double>(r.total) / r.elapsed_seconds : 0.0));
    kv("seed_lookups", u(s.seed_lookups));
    kv("seeds_skipped_n", u(s.seeds_skipped_n));
    kv("seeds_skipped_popular", u(s.seeds_skipped_popular));
    kv("reads_too_short", u(s.reads_too_short));
    kv("distance_calls", u(s.distance_calls));
    kv("distance_calls_after_first", u(s.distance_calls_after_first));
    kv("early_out_after_first", u(s.early_out_after_first));
    if (s.distance_calls_after_first > 0)
        kv("early_out_rate_after_first", fixed4(static_cast<double>(s.early_out_after_first) /
                                                static_cast<double>(s.distance_calls_after_first)));
    else
        kv("early_out_rate_after_first", "na");
    if (s.single_hits > 0)
        kv("first_scored_was_best_rate",
           fixed4(static_cast<double>(s.first_scored_was_best) / static_cast<double>(s.single_hits)));
    else
        kv("first_scored_was_best_rate", "na");
    kv("multi_early_exits", u(s.multi_early_exits));
    kv("pruning_exits", u(s.pruning_exits));
    kv("dp_cells", u(s.dp_cells));
    return o;
}

void add_stats(sa_stats& d, const sa_stats& s) {
    uint64_t* a = reinterpret_cast<uint64_t*>(&d);
    const uint64_t* b = reinterpret_cast<const uint64_t*>(&s);
    for (size_t i = 0; i < sizeof(sa_stats) / 8; ++i) a[i] += b[i];
}

int ctx_fail(sa_context* ctx, int code) { return fail_thread(code, sa_last_error(ctx)); }

}  // namespace

extern "C" {

void sa_default_align_options(sa_align_options* o) {  // REF include/seedaln/driver.hpp:21-32
    std::memset(o, 0, sizeof(*o));
    sa_default_params(&o->params);
    o->threads = 1;
    o->chunk_min_bytes = 4ull << 20;
    o->stable_order = 0;
    o->tolerance = 50;
    o->command_line = "seedaln align";
    o->verify_index = 1;
}

int sa_report_text(const sa_eval_report* r, char* out, uint64_t cap, uint64_t* len) {
    if (!r) return fail_thread(SA_EINVAL, "null report");
    const std::string t = report_text(*r);
    if (len) *len = t.size();
    if (out && cap) {
        const size_t n = std::min<size_t>(cap - 1, t.size());
        std::memcpy(out, t.data(), n);
        out[n] = '\0';
    }
    return SA_OK;
}

int sa_run_index(const char* fasta_path, const char* index_path, int32_t seed_size, int32_t format,
                 int32_t device) {  // REF src/driver.cpp:37-45
    if (!fasta_path || !index_path) return fail_thread(SA_EINVAL, "null argument");
    sa_genome* g = nullptr;
    if (int rc = sa_genome_from_fasta(fasta_path, &g)) return rc;
    const int rc = sa_index_write(g, seed_size, format, device, index_path);
    sa_genome_free(g);
    return rc;
}

int sa_run_align(const sa_align_options* opt, sa_eval_report* report) {
    if (!opt || !opt->index_path || !opt->fastq_path || !opt->output_path)
        return fail_thread(SA_EINVAL, "null argument");
    if (int rc = sa_validate_params(&opt->params)) return rc;  // REF driver.cpp:48
    sa_genome* g_raw = nullptr;
    sa_context* ctx = nullptr;
    // REF driver.cpp:50-55: load the index, then the seed-size check
    if (int rc = sa_index_load(opt->index_path, opt->devices, opt->n_devices, opt->verify_index, &g_raw, &ctx))
        return rc;
    std::unique_ptr<sa_genome, void (*)(sa_genome*)> g(g_raw, sa_genome_free);
    std::unique_ptr<sa_context, void (*)(sa_context*)> cx(ctx, sa_destroy);
    {
        int32_t s = 0;
        sa_index_seed_size(ctx, &s);
        if (s != opt->params.seed_size)
            return fail_thread(SA_EFORMAT, "index was built with seed size " + std::to_string(s) +
                                               ", but --seed-size is " + std::to_string(opt->params.seed_size));
    }
    // REF driver.cpp:57-67: FASTQ size and first-record check
    struct stat sb;
    if (stat(opt->fastq_path, &sb) != 0) return fail_thread(SA_EIO, std::string("cannot stat ") + opt->fastq_path);
    const uint64_t file_size = static_cast<uint64_t>(sb.st_size);
    InFile in(opt->fastq_path);
    if (!in.ok()) return fail_thread(SA_EIO, std::string("cannot open ") + opt->fastq_path + " for reading");
    if (file_size > 0 && find_record_start(in.fd(), 0, file_size) != 0)
        return fail_thread(SA_EPARSE, std::string(opt->fastq_path) + " does not start with a FASTQ record");
    FILE* out = fopen(opt->output_path, "wb");
    if (!out) return fail_thread(SA_EIO, std::string("cannot open ") + opt->output_path + " for writing");
    std::unique_ptr<FILE, int (*)(FILE*)> out_guard(out, fclose);
    const std::string header = sam_header(*g, opt->command_line);
    fwrite(header.data(), 1, header.size(), out);

    const unsigned workers = opt->threads != 0 ? opt->threads : std::max(1u, std::thread::hardware_concurrency());
    if (opt->chunk_min_bytes < 1) return fail_thread(SA_EINVAL, "min_chunk must be >= 1");
    // ChunkScheduler (REF src/scheduler.cpp:8-31), precomputed: the chunk
    // list depends only on the file size, worker count and minimum
    std::vector<std::pair<uint64_t, uint64_t>> chunks;
    for (uint64_t cur = 0; cur < file_size;) {
        uint64_t size = (file_size - cur) / (2 * static_cast<uint64_t>(workers));
        size = std::max<uint64_t>(size, opt->chunk_min_bytes);
        size = std::min<uint64_t>(size, file_size - cur);
        chunks.push_back({cur, cur + size});
        cur += size;
    }

    std::mutex out_mu, fail_mu, rep_mu;
    std::map<size_t, std::string> pending;  // stable order: by chunk index
    size_t next_expected = 0;
    bool write_failed = false;
    auto emit = [&](size_t ci, std::string&& buf) {
        std::lock_guard<std::mutex> lock(out_mu);
        if (!opt->stable_order) {
            write_failed |= fwrite(buf.data(), 1, buf.size(), out) != buf.size();
            return;
        }
        pending.emplace(ci, std::move(buf));
        while (!pending.empty() && pending.begin()->first == next_expected) {
            const std::string& b = pending.begin()->second;
            write_failed |= fwrite(b.data(), 1, b.size(), out) != b.size();
            pending.erase(pending.begin());
            ++next_expected;
        }
    };
    std::atomic<size_t> cursor{0};
    std::atomic<bool> failed{false};
    Error failure{SA_OK, ""};
    Report total;
    sa_stats stats_total;
    std::memset(&stats_total, 0, sizeof(stats_total));

    auto worker = [&]() {
        Report local;
        sa_stats local_stats;
        std::memset(&local_stats, 0, sizeof(local_stats));
        std::vector<sa_result> res;
        try {
            for (;;) {
                if (failed.load()) break;
                const size_t ci = cursor.fetch_add(1);
                if (ci >= chunks.size()) break;
                Reads rd;
                const uint64_t start = find_record_start(in.fd(), chunks[ci].first, file_size);
                if (start < chunks[ci].second) parse_chunk(in.fd(), start, chunks[ci].second, rd);
                const uint64_t n = rd.name_off.size() - 1;
                std::string buf;
                if (n > 0) {
                    res.resize(n);
                    sa_stats st;
                    std::memset(&st, 0, sizeof(st));
                    if (int rc = sa_align_batch(ctx, &opt->params, rd.bases.data(), rd.base_off.data(), n, res.data(),
                                                &st))
                        throw Error{rc, sa_last_error(ctx)};
                    add_stats(local_stats, st);
                    buf.reserve(n * 64 + rd.bases.size() * 2 + rd.names.size());
                    for (uint64_t i = 0; i < n; ++i) {
                        const std::string_view name(rd.names.data() + rd.name_off[i],
                                                    rd.name_off[i + 1] - rd.name_off[i]);
                        const std::string_view bases(rd.bases.data() + rd.base_off[i],
                                                     rd.base_off[i + 1] - rd.base_off[i]);
                        const std::string_view quals(rd.quals.data() + rd.base_off[i],
                                                     rd.base_off[i + 1] - rd.base_off[i]);
                        const sa_result& r = res[i];
                        // REF driver.cpp:114-118 truth scoring (eval.cpp:12-33)
                        std::optional<Score> score;
                        if (auto t = decode_truth(name)) {
                            if (r.kind != SA_SINGLE_HIT) {
                                score = kNotConfident;
                            } else {
                                const size_t c = g->contig_of(r.position);
                                const uint64_t off = r.position - g->contigs[c].start;
                                if (g->contigs[c].name != t->contig || r.direction != t->direction) {
                                    score = kWrong;
                                } else {
                                    const uint64_t d = off > t->position ? off - t->position : t->position - off;
                                    score = d <= opt->tolerance ? kCorrect : kWrong;
                                }
                            }
                        }
                        local.add(r.kind, score);
                        format_record(buf, *g, r, name, bases, quals);
                    }
                }
                emit(ci, std::move(buf));
            }
        } catch (const Error& e) {
            std::lock_guard<std::mutex> lock(fail_mu);
            if (!failed.exchange(true)) failure = e;
        } catch (const std::exception& e) {
            std::lock_guard<std::mutex> lock(fail_mu);
            if (!failed.exchange(true)) failure = Error{SA_ERUNTIME, e.what()};
        }
        std::lock_guard<std::mutex> lock(rep_mu);
        total.merge(local);
        add_stats(stats_total, local_stats);
    };
    const auto t_start = std::chrono::steady_clock::now();  // REF driver.cpp:139: workers only
    if (workers == 1) {
        worker();
    } else {
        std::vector<std::thread> th;
        th.reserve(workers);
        for (unsigned i = 0; i < workers; ++i) th.emplace_back(worker);
        for (auto& t : th) t.join();
    }
    if (failed.load()) return fail_thread(failure.code, failure.msg);
    if (write_failed || fflush(out) != 0)
        return fail_thread(SA_EIO, std::string("failed writing ") + opt->output_path);
    const double elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    sa_eval_report rep;
    std::memset(&rep, 0, sizeof(rep));
    rep.total = total.total;
    rep.single = total.single;
    rep.multiple = total.multiple;
    rep.notfound = total.notfound;
    rep.correct = total.correct;
    rep.wrong = total.wrong;
    rep.no_truth = total.no_truth;
    rep.elapsed_seconds = elapsed;
    rep.stats = stats_total;
    if (opt->report_path && opt->report_path[0]) {
        FILE* rf = fopen(opt->report_path, "wb");
        if (!rf) return fail_thread(SA_EIO, std::string("cannot open ") + opt->report_path + " for writing");
        const std::string t = report_text(rep);
        const bool ok = fwrite(t.data(), 1, t.size(), rf) == t.size();
        fclose(rf);
        if (!ok) return fail_thread(SA_EIO, std::string("failed writing ") + opt->report_path);
    }
    if (report) *report = rep;
    return SA_OK;
}

}  // extern "C"
