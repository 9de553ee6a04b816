// genome_io.cpp -- genome and index files on the host side of the C ABI.
//
//   sa_genome_from_fasta   PackedGenome::from_fasta   (REF src/genome.cpp:48-94)
//   sa_genome_*            PackedGenome accessors, checksum (REF genome.cpp:158-179)
//   sa_index_write         run_index + save_index_file (REF src/driver.cpp:37-45,
//                          src/seed_index.cpp:145-170): the CSR tables are built
//                          on the GPU (csr.cu), the file is byte-identical to the
//                          reference's; or the compact GPU-native SNAPGPU1 file
//                          (genome only -- the GPU rebuilds its index in seconds)
//   sa_index_load          load_index_file (REF src/seed_index.cpp:173-228): same
//                          checks, messages and error class, then the GPU index
//                          is built from the embedded genome and (verify != 0) the
//                          file's tables are checked against a GPU rebuild.
#include <cuda_runtime.h>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "device_index.h"
#include "host_common.h"

static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "index files are little-endian");

using sab::fail_thread;

namespace {

constexpr char kMagic[8] = {'S', 'N', 'A', 'P', 'I', 'D', 'X', '1'};     // REF seed_index.cpp:15
constexpr char kEndMarker[8] = {'S', 'N', 'A', 'P', 'E', 'N', 'D', '1'};  // REF seed_index.cpp:16
constexpr char kGpuMagic[8] = {'S', 'N', 'A', 'P', 'G', 'P', 'U', '1'};   // this library's compact file
constexpr uint32_t kFormatVersion = 1;                                     // REF seed_index.hpp:68
constexpr uint64_t kSaneLimit = uint64_t{1} << 40;                         // REF seed_index.cpp:188

struct FileCloser {
    void operator()(FILE* f) const {
        if (f) fclose(f);
    }
};
using File = std::unique_ptr<FILE, FileCloser>;

struct FormatError {
    std::string msg;
};

class Reader {  // little-endian reads that fail as the reference's get<> does
public:
    explicit Reader(FILE* f) : f_(f) {}
    template <typename T>
    T get() {
        T v;
        if (fread(&v, sizeof(T), 1, f_) != 1) throw FormatError{"truncated index file"};
        return v;
    }
    void bytes(void* dst, size_t n, const char* what = "truncated index file") {
        if (n && fread(dst, 1, n, f_) != n) throw FormatError{what};
    }
    std::vector<uint64_t> words() {
        const uint64_t n = get<uint64_t>();
        if (n > kSaneLimit) throw FormatError{"corrupt index file: bad array size"};
        std::vector<uint64_t> w;
        // grow in bounded steps so a corrupt count cannot allocate beyond the file
        const uint64_t step = uint64_t{1} << 24;
        for (uint64_t done = 0; done < n;) {
            const uint64_t k = std::min(step, n - done);
            w.resize(done + k);
            bytes(w.data() + done, k * sizeof(uint64_t));
            done += k;
        }
        return w;
    }

private:
    FILE* f_;
};

class Writer {
public:
    explicit Writer(FILE* f) : f_(f) {}
    template <typename T>
    void put(T v) {
        ok_ &= fwrite(&v, sizeof(T), 1, f_) == 1;
    }
    void bytes(const void* p, size_t n) {
        if (n) ok_ &= fwrite(p, 1, n, f_) == n;
    }
    void words(const std::vector<uint64_t>& w) {
        put<uint64_t>(w.size());
        bytes(w.data(), w.size() * sizeof(uint64_t));
    }
    bool ok() const { return ok_; }

private:
    FILE* f_;
    bool ok_ = true;
};

void write_genome(Writer& w, const sa_genome& g) {  // REF seed_index.cpp:154-163
    w.put<uint64_t>(g.contigs.size());
    for (const auto& c : g.contigs) {
        w.put<uint32_t>(static_cast<uint32_t>(c.name.size()));
        w.bytes(c.name.data(), c.name.size());
        w.put<uint64_t>(c.start);
        w.put<uint64_t>(c.length);
    }
    w.put<uint64_t>(g.length);
    w.words(g.packed);
    w.words(g.nmask);
}

void read_genome(Reader& r, sa_genome& g) {  // REF seed_index.cpp:188-205
    const uint64_t contig_count = r.get<uint64_t>();
    if (contig_count > kSaneLimit) throw FormatError{"corrupt index file"};
    g.contigs.clear();
    for (uint64_t i = 0; i < contig_count; ++i) {
        sa_genome::Contig c;
        const uint32_t len = r.get<uint32_t>();
        c.name.resize(len);
        r.bytes(c.name.data(), len);
        c.start = r.get<uint64_t>();
        c.length = r.get<uint64_t>();
        g.contigs.push_back(std::move(c));
    }
    g.length = r.get<uint64_t>();
    g.packed = r.words();
    g.nmask = r.words();
    if (g.packed.size() != (g.length + 31) / 32 || g.nmask.size() != (g.length + 63) / 64)
        throw FormatError{"corrupt index file: genome size mismatch"};
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail_thread(SA_ERUNTIME, std::string(what) + ": " + cudaGetErrorString(e));
}

// CSR tables of g on `device` (csr.cu).
int gpu_csr(const sa_genome& g, int s, int device, sab::CsrIndex& csr) {
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    cudaStream_t st = nullptr;
    if ((e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess)
        return cuda_fail(e, "cudaStreamCreate");
    uint4* planes = nullptr;
    std::string err;
    int rc = sab::upload_planes(g.packed.data(), g.packed.size(), g.nmask.data(), g.nmask.size(), g.length, st,
                                &planes, err);
    if (rc == 0) rc = sab::build_csr_index(planes, g.length, s, st, &csr, err);
    if (planes) cudaFree(planes);
    cudaStreamDestroy(st);
    if (rc) return fail_thread(rc == 1 ? SA_EINVAL : SA_ERUNTIME, "GPU CSR build: " + err);
    return SA_OK;
}

}  // namespace

// ---------------------------------------------------------------- sa_genome

uint64_t sa_genome::checksum() const {  // REF src/genome.cpp:158-179, FNV-1a
    uint64_t h = 14695981039346656037ull;
    auto mix = [&h](uint64_t v) {
        for (int i = 0; i < 8; ++i) {
            h ^= (v >> (i * 8)) & 0xff;
            h *= 1099511628211ull;
        }
    };
    mix(length);
    for (const Contig& c : contigs) {
        for (char ch : c.name) {
            h ^= static_cast<unsigned char>(ch);
            h *= 1099511628211ull;
        }
        mix(c.start);
        mix(c.length);
    }
    for (uint64_t w : packed) mix(w);
    for (uint64_t w : nmask) mix(w);
    return h;
}

size_t sa_genome::contig_of(uint64_t pos) const {
    auto it = std::upper_bound(contigs.begin(), contigs.end(), pos,
                               [](uint64_t p, const Contig& c) { return p < c.start; });
    return static_cast<size_t>(it - contigs.begin()) - 1;
}

namespace sab {

int char_to_code(char c) {
    const char u = static_cast<char>(std::toupper(static_cast<unsigned char>(c)));
    switch (u) {
        case 'A': return 0;
        case 'C': return 1;
        case 'G': return 2;
        case 'T': return 3;
        default:
            return std::strchr("ACGTUNRYSWKMBDHV", u) != nullptr && u != '\0' ? 4 : -1;
    }
}

}  // namespace sab

extern "C" {

int sa_genome_from_fasta(const char* path, sa_genome** out) {
    if (!out || !path) return fail_thread(SA_EINVAL, "null argument");
    *out = nullptr;
    File f(fopen(path, "rb"));
    if (!f) return fail_thread(SA_EIO, std::string("cannot open ") + path + " for reading");
    auto g = std::make_unique<sa_genome>();
    bool have_contig = false;
    size_t line_no = 0;
    auto close_contig = [&] {
        if (have_contig) g->contigs.back().length = g->length - g->contigs.back().start;
    };
    std::vector<char> buf(1 << 22);
    std::string line;
    // getline semantics over a block reader (REF genome.cpp:56-91)
    size_t have = 0, at = 0;
    bool eof = false;
    auto next_line = [&](std::string& l) -> bool {
        l.clear();
        for (;;) {
            if (at == have) {
                if (eof) return !l.empty();
                have = fread(buf.data(), 1, buf.size(), f.get());
                at = 0;
                if (have == 0) {
                    eof = true;
                    return !l.empty();
                }
            }
            const char* s = buf.data() + at;
            const char* nl = static_cast<const char*>(std::memchr(s, '\n', have - at));
            if (nl) {
                l.append(s, nl - s);
                at += (nl - s) + 1;
                return true;
            }
            l.append(s, have - at);
            at = have;
        }
    };
    while (next_line(line)) {
        ++line_no;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty()) continue;
        if (line[0] == '>') {
            close_contig();
            std::string name = line.substr(1);
            const size_t ws = name.find_first_of(" \t");
            if (ws != std::string::npos) name.resize(ws);
            if (name.empty())
                return fail_thread(SA_EPARSE, "FASTA header with empty name at line " + std::to_string(line_no));
            g->contigs.push_back({std::move(name), g->length, 0});
            have_contig = true;
            continue;
        }
        if (!have_contig)
            return fail_thread(SA_EPARSE, "FASTA sequence before any '>' header at line " + std::to_string(line_no));
        for (char c : line) {
            if (std::isspace(static_cast<unsigned char>(c))) continue;
            const int code = sab::char_to_code(c);
            if (code < 0)
                return fail_thread(SA_EPARSE, std::string("illegal FASTA character '") + c + "' at line " +
                                                  std::to_string(line_no));
            g->append(code);
        }
    }
    if (ferror(f.get())) return fail_thread(SA_EIO, std::string("failed reading ") + path);
    close_contig();
    if (g->contigs.empty()) return fail_thread(SA_EPARSE, "empty FASTA input");
    *out = g.release();
    return SA_OK;
}

int sa_genome_from_words(const uint64_t* packed, uint64_t n_packed, const uint64_t* nmask, uint64_t n_nmask,
                         uint64_t length, const char* const* names, const uint64_t* starts,
                         const uint64_t* lengths, uint64_t n_contigs, sa_genome** out) {
    if (!out) return fail_thread(SA_EINVAL, "null argument");
    *out = nullptr;
    if (n_packed != (length + 31) / 32 || n_nmask != (length + 63) / 64)
        return fail_thread(SA_EFORMAT, "packed/n-mask word counts do not match genome length");
    if ((n_packed && !packed) || (n_nmask && !nmask) || (n_contigs && (!names || !starts || !lengths)))
        return fail_thread(SA_EINVAL, "null argument");
    auto g = std::make_unique<sa_genome>();
    g->length = length;
    g->packed.assign(packed, packed + n_packed);
    g->nmask.assign(nmask, nmask + n_nmask);
    for (uint64_t i = 0; i < n_contigs; ++i) g->contigs.push_back({names[i], starts[i], lengths[i]});
    *out = g.release();
    return SA_OK;
}

void sa_genome_free(sa_genome* g) { delete g; }

int sa_genome_info(const sa_genome* g, uint64_t* length, uint64_t* n_contigs, uint64_t* checksum) {
    if (!g) return fail_thread(SA_EINVAL, "null genome");
    if (length) *length = g->length;
    if (n_contigs) *n_contigs = g->contigs.size();
    if (checksum) *checksum = g->checksum();
    return SA_OK;
}

int sa_genome_words(const sa_genome* g, const uint64_t** packed, uint64_t* n_packed, const uint64_t** nmask,
                    uint64_t* n_nmask) {
    if (!g) return fail_thread(SA_EINVAL, "null genome");
    if (packed) *packed = g->packed.data();
    if (n_packed) *n_packed = g->packed.size();
    if (nmask) *nmask = g->nmask.data();
    if (n_nmask) *n_nmask = g->nmask.size();
    return SA_OK;
}

int sa_genome_contig(const sa_genome* g, uint64_t i, const char** name, uint64_t* start, uint64_t* length) {
    if (!g) return fail_thread(SA_EINVAL, "null genome");
    if (i >= g->contigs.size()) return fail_thread(SA_EINVAL, "contig index out of range");
    if (name) *name = g->contigs[i].name.c_str();
    if (start) *start = g->contigs[i].start;
    if (length) *length = g->contigs[i].length;
    return SA_OK;
}

int sa_create_from_genome(const sa_genome* g, int32_t seed_size, const int32_t* devices, int32_t n_devices,
                          sa_context** out) {
    if (!g) return fail_thread(SA_EINVAL, "null genome");
    return sa_create(g->packed.data(), g->packed.size(), g->nmask.data(), g->nmask.size(), g->length, seed_size,
                     devices, n_devices, out);
}

int sa_index_write(const sa_genome* g, int32_t seed_size, int32_t format, int32_t device, const char* path) {
    if (!g || !path) return fail_thread(SA_EINVAL, "null argument");
    if (seed_size < 1 || seed_size > 32)  // REF seed_index.cpp:81-82
        return fail_thread(SA_EINVAL, "seed size must be in [1, 32]");
    if (g->length < static_cast<uint64_t>(seed_size))  // REF :83-84
        return fail_thread(SA_EINVAL, "genome shorter than seed size");
    if (format != SA_INDEX_SNAPIDX1 && format != SA_INDEX_SNAPGPU1)
        return fail_thread(SA_EINVAL, "unknown index file format");
    sab::CsrIndex csr;
    if (format == SA_INDEX_SNAPIDX1) {
        if (int rc = gpu_csr(*g, seed_size, device, csr)) return rc;
    }
    File f(fopen(path, "wb"));
    if (!f) return fail_thread(SA_EIO, std::string("cannot open ") + path + " for writing");
    Writer w(f.get());
    // REF seed_index.cpp:150-169
    w.bytes(format == SA_INDEX_SNAPIDX1 ? kMagic : kGpuMagic, 8);
    w.put<uint32_t>(kFormatVersion);
    w.put<uint32_t>(static_cast<uint32_t>(seed_size));
    w.put<uint64_t>(g->checksum());
    write_genome(w, *g);
    if (format == SA_INDEX_SNAPIDX1) {
        w.words(csr.keys);
        w.words(csr.offsets);
        w.words(csr.positions);
    }
    w.bytes(kEndMarker, 8);
    if (!w.ok() || fflush(f.get()) != 0) return fail_thread(SA_EIO, std::string("failed writing ") + path);
    return SA_OK;
}

int sa_index_load(const char* path, const int32_t* devices, int32_t n_devices, int32_t verify,
                  sa_genome** genome_out, sa_context** ctx_out) {
    if (!path || !genome_out || !ctx_out) return fail_thread(SA_EINVAL, "null argument");
    *genome_out = nullptr;
    *ctx_out = nullptr;
    File f(fopen(path, "rb"));
    if (!f) return fail_thread(SA_EIO, std::string("cannot open ") + path + " for reading");
    auto g = std::make_unique<sa_genome>();
    int seed_size = 0;
    bool gpu_file = false;
    sab::CsrIndex file_csr;
    uint64_t stored_checksum = 0;
    try {  // REF seed_index.cpp:173-228, same order of checks and messages
        Reader r(f.get());
        char magic[8];
        r.bytes(magic, 8, "not a seed index file (bad magic)");
        gpu_file = std::equal(magic, magic + 8, kGpuMagic);
        if (!gpu_file && !std::equal(magic, magic + 8, kMagic))
            throw FormatError{"not a seed index file (bad magic)"};
        const uint32_t version = r.get<uint32_t>();
        if (version != kFormatVersion)
            throw FormatError{"index format version mismatch: file has " + std::to_string(version) +
                              ", expected " + std::to_string(kFormatVersion)};
        seed_size = static_cast<int>(r.get<uint32_t>());
        if (seed_size < 1 || seed_size > 32) throw FormatError{"corrupt index file: bad seed size"};
        stored_checksum = r.get<uint64_t>();
        read_genome(r, *g);
        if (!gpu_file) {
            file_csr.keys = r.words();
            file_csr.offsets = r.words();
            file_csr.positions = r.words();
            if (file_csr.offsets.size() != file_csr.keys.size() + 1 ||
                (file_csr.offsets.empty() ? 0 : file_csr.offsets.back()) != file_csr.positions.size())
                throw FormatError{"corrupt index file: inconsistent tables"};
        }
        char marker[8];
        r.bytes(marker, 8);
        if (!std::equal(marker, marker + 8, kEndMarker)) throw FormatError{"truncated index file"};
        if (g->checksum() != stored_checksum) throw FormatError{"genome checksum mismatch"};
    } catch (const FormatError& e) {
        return fail_thread(SA_EFORMAT, e.msg);
    }
    f.reset();
    if (verify && !gpu_file) {
        // The reference would use the stored tables as they are; here the GPU
        // builds its own index from the embedded genome, so the tables must be
        // the genome's index -- true for every file save_index_file writes.
        sab::CsrIndex mine;
        const int dev = devices && n_devices > 0 ? devices[0] : 0;
        if (int rc = gpu_csr(*g, seed_size, dev, mine)) return rc;
        if (mine.keys != file_csr.keys || mine.offsets != file_csr.offsets || mine.positions != file_csr.positions)
            return fail_thread(SA_EFORMAT, "index tables do not match the embedded genome");
    }
    file_csr = sab::CsrIndex{};
    sa_context* ctx = nullptr;
    if (int rc = sa_create_from_genome(g.get(), seed_size, devices, n_devices, &ctx)) return rc;
    *ctx_out = ctx;
    *genome_out = g.release();
    return SA_OK;
}

int sa_index_csr(const sa_genome* g, int32_t seed_size, int32_t device, uint64_t* n_keys, uint64_t* n_positions,
                 uint64_t* keys, uint64_t* offsets, uint64_t* positions) {
    if (!g || !n_keys || !n_positions) return fail_thread(SA_EINVAL, "null argument");
    if (seed_size < 1 || seed_size > 32) return fail_thread(SA_EINVAL, "seed size must be in [1, 32]");
    if (g->length < static_cast<uint64_t>(seed_size)) return fail_thread(SA_EINVAL, "genome shorter than seed size");
    sab::CsrIndex csr;
    if (int rc = gpu_csr(*g, seed_size, device, csr)) return rc;
    const uint64_t cap_k = *n_keys, cap_p = *n_positions;
    *n_keys = csr.keys.size();
    *n_positions = csr.positions.size();
    if (keys && offsets && positions) {
        if (cap_k < csr.keys.size() || cap_p < csr.positions.size())
            return fail_thread(SA_EINVAL, "output arrays too small");
        std::copy(csr.keys.begin(), csr.keys.end(), keys);
        std::copy(csr.offsets.begin(), csr.offsets.end(), offsets);
        std::copy(csr.positions.begin(), csr.positions.end(), positions);
    }
    return SA_OK;
}

}  // extern "C"
