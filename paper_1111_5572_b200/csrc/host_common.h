// host_common.h -- host-side shared pieces of the C-ABI library.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/snap_b200.h"

// PackedGenome (REF include/seedaln/genome.hpp:36-100): 2-bit words
// (32 bases per word, LSB-first), an N bitmask (64 positions per word) and the
// contig table tiling [0, length) in file order.
struct sa_genome {
    struct Contig {
        std::string name;
        uint64_t start = 0, length = 0;
    };
    uint64_t length = 0;
    std::vector<uint64_t> packed, nmask;
    std::vector<Contig> contigs;

    // REF src/genome.cpp:39-46 append_base
    void append(int code) {  // 0..3 = ACGT, 4 = N
        const uint64_t pos = length++;
        if ((pos & 31) == 0) packed.push_back(0);
        if ((pos & 63) == 0) nmask.push_back(0);
        packed[pos >> 5] |= static_cast<uint64_t>(code == 4 ? 0 : code) << ((pos & 31) * 2);
        if (code == 4) nmask[pos >> 6] |= uint64_t{1} << (pos & 63);
    }
    uint64_t checksum() const;
    // REF src/genome.cpp:121-131: last contig whose start <= pos
    size_t contig_of(uint64_t pos) const;
};

namespace sab {

void set_thread_error(const std::string& msg);
int fail_thread(int code, const std::string& msg);

// REF src/genome.cpp:23-37 char_to_base: ACGT any case -> 0..3, IUPAC -> 4,
// anything else -> -1.
int char_to_code(char c);

// pack.cpp: ASCII reads -> three bit planes {lo, hi, n} (host thread pool)
bool pack_enabled(bool pageable);  // host packing of this call's reads (pack.cpp)
uint64_t pack_words_per_plane(uint64_t n_bases);
void pack_planar(const char* src, uint64_t n, uint32_t* planes, uint64_t wpp);
// multi-threaded memcpy (host thread pool), for staging pageable input
void parallel_copy(void* dst, const void* src, uint64_t n);

}  // namespace sab
