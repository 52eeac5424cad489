// AERO binary stream files (reference streams.cpp:105-137 load_aero,
// :150-168 save_stream): "AERO", version byte 0x01, u32 d, u64 n (0 = until
// EOF), then n rows of d little-endian fp64, row-major.
//
// The reference loads a whole file into memory before any update. The
// configs' inputs do not fit that (C2 32 GB, C4 128 GB per site), so here a
// file is STREAMED: a reader thread fills two pinned host buffers in turn
// while the sketch absorbs the previous chunk (its H2D is a DMA from pinned
// memory inside update_block's own double-buffered staging). Validation keeps
// the reference's FormatError cases (bad magic or version, truncated header,
// zero dimension, truncated row, non-finite value); a chunk is checked before
// it is absorbed, so rows of earlier chunks are already in the sketch when a
// later chunk raises (the reference raises before any update).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "aero_common.cuh"
#include "aeroio.hpp"
#include "sketch.hpp"

namespace aero_b200 {

static_assert(sizeof(double) == 8, "AERO rows are 8-byte doubles");
namespace {
constexpr unsigned char kMagic[4] = {0x41, 0x45, 0x52, 0x4f};  // "AERO"
constexpr unsigned char kVersion = 0x01;
}  // namespace

AeroFile::AeroFile(const std::string& path) : path_(path) {
    f_ = std::fopen(path.c_str(), "rb");
    if (!f_) throw FormatError("cannot open " + path);
    unsigned char hdr[17];
    const size_t got = std::fread(hdr, 1, sizeof(hdr), f_);
    if (got < 4 || std::memcmp(hdr, kMagic, 4) != 0) {
        std::fclose(f_);
        f_ = nullptr;
        throw FormatError(path + ": bad magic");
    }
    if (got < 5 || hdr[4] != kVersion) {
        std::fclose(f_);
        f_ = nullptr;
        throw FormatError(path + ": unsupported version");
    }
    if (got < 17) {
        std::fclose(f_);
        f_ = nullptr;
        throw FormatError(path + ": truncated header");
    }
    std::memcpy(&d_, hdr + 5, 4);
    std::memcpy(&n_, hdr + 9, 8);
    if (d_ == 0) {
        std::fclose(f_);
        f_ = nullptr;
        throw FormatError(path + ": zero dimension");
    }
}
AeroFile::~AeroFile() {
    if (f_) std::fclose(f_);
}

// next rows into out (max_rows x d); returns the count (0 at the end)
int64_t AeroFile::read(double* out, int64_t max_rows) {
    int64_t k = 0;
    const size_t row_bytes = (size_t)8 * d_;
    while (k < max_rows && (n_ == 0 || read_ < n_)) {
        const size_t got = std::fread(out + (size_t)k * d_, 1, row_bytes, f_);
        if (got != row_bytes) {
            if (n_ == 0 && got == 0) {  // n = 0: until EOF
                done_ = true;
                break;
            }
            throw FormatError(path_ + ": truncated row " + std::to_string(read_ + 1));
        }
        const double* r = out + (size_t)k * d_;
        for (uint32_t j = 0; j < d_; ++j)
            if (!std::isfinite(r[j])) throw FormatError(path_ + ": non-finite value");
        ++read_;
        ++k;
    }
    if (n_ > 0 && read_ >= n_) done_ = true;
    return k;
}

void aero_file_write(const std::string& path, const double* rows, int64_t n, int d) {
    if (n < 1) throw InvalidInput("save_stream: empty record set");
    if (d < 1) throw InvalidInput("save_stream: nonuniform dimension");
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw FormatError("cannot write " + path);
    const uint32_t d32 = (uint32_t)d;
    const uint64_t n64 = (uint64_t)n;
    bool ok = std::fwrite(kMagic, 1, 4, f) == 4 && std::fwrite(&kVersion, 1, 1, f) == 1 &&
              std::fwrite(&d32, 4, 1, f) == 1 && std::fwrite(&n64, 8, 1, f) == 1 &&
              std::fwrite(rows, 8, (size_t)n * d, f) == (size_t)n * d;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw FormatError("write failure on " + path);
}

// Stream a file through a sketch: chunk k+1 is read from disk (reader thread,
// pinned buffer) while chunk k is absorbed. Row q of the file has timestamp
// t0 + q (StreamRecord::t is 1-based and contiguous, streams.hpp:20-24).
int64_t aero_file_update(Sketch& s, const std::string& path, int64_t t0, int64_t chunk_rows,
                         aero_event* log, int64_t log_cap) {
    AeroFile f(path);
    if ((int)f.d() != s.d()) throw InvalidInput("AeroState: row dimension mismatch");
    if (chunk_rows < 1) chunk_rows = 16384;
    const int d = s.d();
    double* buf[2] = {nullptr, nullptr};
    for (int b = 0; b < 2; ++b) AERO_CUDA(cudaMallocHost(&buf[b], sizeof(double) * (size_t)chunk_rows * d));
    struct Free {
        double** b;
        ~Free() {
            cudaFreeHost(b[0]);
            cudaFreeHost(b[1]);
        }
    } free_bufs{buf};
    int64_t got[2] = {0, 0};
    std::string err[2];
    auto fill = [&](int b) {
        try {
            got[b] = f.read(buf[b], chunk_rows);
        } catch (const std::exception& e) {
            got[b] = -1;
            err[b] = e.what();
        }
    };
    std::vector<int64_t> ts;
    std::vector<aero_event> evs;
    int64_t total = 0;
    fill(0);
    for (int k = 0;; ++k) {
        const int b = k & 1;
        if (got[b] < 0) throw FormatError(err[b]);
        if (got[b] == 0) break;
        std::thread next;
        const bool more = !f.done();
        if (more) next = std::thread(fill, b ^ 1);
        const int64_t m = got[b];
        ts.resize(m);
        for (int64_t q = 0; q < m; ++q) ts[q] = t0 + total + q;
        aero_event* lg = nullptr;
        if (log && total + m <= log_cap) lg = log + total;
        else {
            evs.resize(m);
            lg = evs.data();
        }
        try {
            s.update_block(buf[b], false, m, d, ts.data(), nullptr, lg);
        } catch (...) {
            if (next.joinable()) next.join();
            throw;
        }
        total += m;
        if (next.joinable()) next.join();
        if (!more) break;
    }
    return total;
}

}  // namespace aero_b200
