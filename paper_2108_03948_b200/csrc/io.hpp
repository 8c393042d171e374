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
struct HostSpectrum {
    std::vector<double> bins;   // interleaved re, im
    double f_start = 0.0, f_step = 0.0;
    size_t source_n = 0;
};
// read_spectrum_csv (spectra.cpp:94-150): "frequency_hz,re,im,magnitude_db" rows, optional header,
// uniform axis check; read_spectrum_csv_file (spectra.cpp:152-156), "-" = stdin
HostSpectrum parse_spectrum_csv(const char* data, size_t len, const std::string& origin);
HostSpectrum read_spectrum_csv_file(const std::string& path);
// write_trace_csv (signals.cpp:178-189) to a file ("-" = stdout); validates like the reference
void write_trace_csv_file(const double* samples, size_t n, double fs, double t0, const std::string& path);
// write_spectrum_csv (spectra.cpp:63-72): "frequency_hz,re,im,magnitude_db" + %.17g rows
void write_spectrum_csv_file(const double* bins_interleaved, size_t n, double f_start, double f_step,
                             const std::string& path);
// write_spectrum_json (spectra.cpp:161-183): the reference's JSON object, numbers as its JSON library
// prints them (Grisu2 shortest digits); byte-identical files
std::string format_spectrum_json(const double* bins_interleaved, size_t n, double f_start, double f_step,
                                 size_t source_n);
void write_spectrum_json_file(const double* bins_interleaved, size_t n, double f_start, double f_step,
                              size_t source_n, const std::string& path);
// one double as the reference's JSON library prints it (non-finite: null)
void json_number(std::string& out, double v);
// the CSV body as a string (the same bytes the file gets)
std::string format_spectrum_csv(const double* bins_interleaved, size_t n, double f_start, double f_step);

// open a reference-format output file (serialize.cpp:22-26 message; "-" = stdout), write, close
void write_text_file(const std::string& body, const std::string& path, const char* open_msg, const char* what);
// %.17g of v appended to out (std::to_chars, the printf format the reference uses)
void append_g17(std::string& out, double v);

// run fn(i) for i < count on up to `threads` host threads (0 = all cores); the lowest-index
// exception is rethrown after every task finished
void parallel_for(size_t count, int threads, const std::function<void(size_t)>& fn);

}  // namespace skg
