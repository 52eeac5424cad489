// AERO binary stream files, streamed (aeroio.cu; reference streams.cpp:105-168)
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/aero_b200.h"

namespace aero_b200 {

class Sketch;

class AeroFile {
  public:
    explicit AeroFile(const std::string& path);  // reads and validates the header
    ~AeroFile();
    AeroFile(const AeroFile&) = delete;
    AeroFile& operator=(const AeroFile&) = delete;
    uint32_t d() const { return d_; }
    uint64_t n_header() const { return n_; }  // 0 = rows until EOF
    int64_t read(double* out, int64_t max_rows);
    bool done() const { return done_; }

  private:
    std::string path_;
    std::FILE* f_ = nullptr;
    uint32_t d_ = 0;
    uint64_t n_ = 0, read_ = 0;
    bool done_ = false;
};

void aero_file_write(const std::string& path, const double* rows, int64_t n, int d);
int64_t aero_file_update(Sketch& s, const std::string& path, int64_t t0, int64_t chunk_rows, aero_event* log,
                         int64_t log_cap);

}  // namespace aero_b200
