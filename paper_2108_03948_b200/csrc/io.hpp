// io.hpp — trace ingest and spectrum serialisation on the host side of the batched path
// (SURVEY §8f rows 1-2): the reference's CSV formats restated byte for byte, parallel over files,
// staged through pinned memory to / from the device batch buffers.
#pragma once

#include <cstddef>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace skg {

// the reference's error classes (errors.hpp:9-25); the C ABI maps them to SK_ERR_IO / PARSE / FORMAT
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ParseError : std::runtime_error {
    ParseError(const std::string& m, size_t l) : std::runtime_error(m), line(l) {}
    size_t line = 0;
};
struct FormatError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct HostTrace {
    std::vector<double> samples;
    double fs = 0.0, t0 = 0.0;
};

// read_trace_csv (signals.cpp:125-170) over an in-memory file; `origin` prefixes the messages
HostTrace parse_trace_csv(const char* data, size_t len, const std::string& origin);
// read_trace_csv_file (signals.cpp:172-176); "-" reads stdin (capi.cpp:98, 394)
HostTrace read_trace_csv_file(const std::string& path);
// write_trace_csv (signals.cpp:178-189) to a file ("-" = stdout); validates like the reference
void write_trace_csv_file(const double* samples, size_t n, double fs, double t0, const std::string& path);
// write_spectrum_csv (spectra.cpp:63-72): "frequency_hz,re,im,magnitude_db" + %.17g rows
void write_spectrum_csv_file(const double* bins_interleaved, size_t n, double f_start, double f_step,
                             const std::string& path);
// the CSV body as a string (the same bytes the file gets)
std::string format_spectrum_csv(const double* bins_interleaved, size_t n, double f_start, double f_step);

// run fn(i) for i < count on up to `threads` host threads (0 = all cores); the lowest-index
// exception is rethrown after every task finished
void parallel_for(size_t count, int threads, const std::function<void(size_t)>& fn);

}  // namespace skg
