// io.cpp — trace ingest / spectrum serialisation restated from the reference (signals.cpp:100-189,
// spectra.cpp:63-78) for the batched path: whole-file reads, std::from_chars parsing (the
// reference's own parser), std::to_chars(general, 17) formatting (specified as printf's %.17g, the
// reference's snprintf format, so the bytes are identical), files processed in parallel.
#include "io.hpp"

#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string_view>
#include <thread>

#include "grisu_powers.hpp"

namespace skg {

namespace {

bool parse_double(std::string_view field, double& out) {   // signals.cpp:102-112
    while (!field.empty() && (field.front() == ' ' || field.front() == '\t')) field.remove_prefix(1);
    while (!field.empty() && (field.back() == ' ' || field.back() == '\t')) field.remove_suffix(1);
    if (field.empty()) return false;
    const char* last = field.data() + field.size();
    auto [ptr, ec] = std::from_chars(field.data(), last, out);
    return ec == std::errc{} && ptr == last;
}

bool parse_row(std::string_view line, double& t, double& x) {   // signals.cpp:114-120
    const size_t comma = line.find(',');
    if (comma == std::string_view::npos) return false;
    if (line.find(',', comma + 1) != std::string_view::npos) return false;
    return parse_double(line.substr(0, comma), t) && parse_double(line.substr(comma + 1), x);
}

std::string slurp(FILE* f) {
    std::string s;
    char buf[1 << 16];
    size_t r;
    while ((r = fread(buf, 1, sizeof buf, f)) > 0) s.append(buf, r);
    return s;
}

// %.17g into p (returns the end)
char* put_g17(char* p, char* end, double v) {
    auto r = std::to_chars(p, end, v, std::chars_format::general, 17);
    return r.ptr;
}

double magnitude_db(double re, double im) {   // types.cpp:13-18 (std::abs of std::complex = hypot)
    const double mag = std::hypot(re, im);
    return mag > 1e-15 ? 20.0 * std::log10(mag) : -300.0;
}

FILE* open_out(const std::string& path, const char* what) {
    if (path == "-") return stdout;
    FILE* f = fopen(path.c_str(), "wb");
    if (!f) throw IoError(std::string("cannot open ") + what + " file for writing: " + path);
    return f;
}

void finish_out(FILE* f, bool ok, const char* what) {
    if (f != stdout) ok = (fclose(f) == 0) && ok;
    else ok = (fflush(f) == 0) && ok;
    if (!ok) throw IoError(std::string(what) + ": write failed");
}

// ---- JSON numbers: Grisu2 (Loitsch, "Printing floating-point numbers quickly and accurately with
// integers", PLDI 2010) with the conservative boundaries, then the decimal layout the reference's JSON
// library prints (plain notation for decimal exponents in (-4, 15], else d.ddde+XX; integral values
// keep ".0"). The reference's spectrum JSON (spectra.cpp:161-176) formats every double this way.
namespace grisu {
struct Fp {
    uint64_t f;
    int e;
};
Fp mul(Fp x, Fp y) {   // the upper 64 bits of the 128-bit product, rounded half up
    const unsigned __int128 p = (unsigned __int128)x.f * y.f;
    const uint64_t h = (uint64_t)(p >> 64), l = (uint64_t)p;
    return {h + (l >> 63), x.e + y.e + 64};
}
Fp normalize(Fp x) {
    while ((x.f >> 63) == 0) {
        x.f <<= 1;
        x.e--;
    }
    return x;
}
Fp normalize_to(Fp x, int e) { return {x.f << (x.e - e), e}; }

void boundaries(double value, Fp& w, Fp& lo, Fp& hi) {
    uint64_t bits;
    std::memcpy(&bits, &value, sizeof bits);
    const uint64_t E = bits >> 52, F = bits & ((uint64_t{1} << 52) - 1);
    constexpr int kBias = 1075, kMinExp = 1 - kBias;
    const Fp v = E == 0 ? Fp{F, kMinExp} : Fp{F + (uint64_t{1} << 52), (int)E - kBias};
    const bool lower_closer = F == 0 && E > 1;   // the gap below a power of two is half the gap above
    const Fp m_plus{2 * v.f + 1, v.e - 1};
    const Fp m_minus = lower_closer ? Fp{4 * v.f - 1, v.e - 2} : Fp{2 * v.f - 1, v.e - 1};
    hi = normalize(m_plus);
    lo = normalize_to(m_minus, hi.e);
    w = normalize(v);
}

int largest_pow10(uint32_t n, uint32_t& p) {
    static const uint32_t t[] = {1u, 10u, 100u, 1000u, 10000u, 100000u, 1000000u, 10000000u, 100000000u, 1000000000u};
    int k = 10;
    while (k > 1 && n < t[k - 1]) --k;
    p = t[k - 1];
    return k;
}

void round_weed(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ten_k) {
    while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
        buf[len - 1]--;
        rest += ten_k;
    }
}

// shortest-in-practice digits of value > 0: buf[0..len) x 10^dexp
void digits(double value, char* buf, int& len, int& dexp) {
    Fp w, lo, hi;
    boundaries(value, w, lo, hi);
    constexpr int kAlpha = -60;
    const int f = kAlpha - hi.e - 1;
    const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);
    const int index = (-kCachedPowersMinDecExp + k + (kCachedPowersDecStep - 1)) / kCachedPowersDecStep;
    const CachedPow10 c = kCachedPowers[index];
    const Fp ck{c.f, c.e};
    const Fp W = mul(w, ck), Wlo = mul(lo, ck), Whi = mul(hi, ck);
    const Fp Mm{Wlo.f + 1, Wlo.e}, Mp{Whi.f - 1, Whi.e};
    dexp = -c.k;
    len = 0;
    uint64_t delta = Mp.f - Mm.f, dist = Mp.f - W.f;
    const Fp one{uint64_t{1} << -Mp.e, Mp.e};
    uint32_t p1 = (uint32_t)(Mp.f >> -one.e);
    uint64_t p2 = Mp.f & (one.f - 1);
    uint32_t pow10;
    int n = largest_pow10(p1, pow10);
    while (n > 0) {
        const uint32_t d = p1 / pow10, r = p1 % pow10;
        buf[len++] = (char)('0' + d);
        p1 = r;
        n--;
        const uint64_t rest = (uint64_t{p1} << -one.e) + p2;
        if (rest <= delta) {
            dexp += n;
            round_weed(buf, len, dist, delta, rest, uint64_t{pow10} << -one.e);
            return;
        }
        pow10 /= 10;
    }
    int m = 0;
    for (;;) {
        p2 *= 10;
        const uint64_t d = p2 >> -one.e, r = p2 & (one.f - 1);
        buf[len++] = (char)('0' + d);
        p2 = r;
        m++;
        delta *= 10;
        dist *= 10;
        if (p2 <= delta) break;
    }
    dexp -= m;
    round_weed(buf, len, dist, delta, p2, one.f);
}
}  // namespace grisu

// one finite double as the reference's JSON library prints it
void append_json_number(std::string& out, double v) {
    if (!std::isfinite(v)) {
        out += "null";
        return;
    }
    if (std::signbit(v)) {
        out += '-';
        v = -v;
    }
    if (v == 0.0) {
        out += "0.0";
        return;
    }
    char d[32];
    int k = 0, dexp = 0;
    grisu::digits(v, d, k, dexp);
    const int n = k + dexp;   // decimal point position relative to the digits
    constexpr int kMin = -4, kMax = 15;
    if (k <= n && n <= kMax) {   // digits000.0
        out.append(d, k);
        out.append((size_t)(n - k), '0');
        out += ".0";
    } else if (0 < n && n <= kMax) {   // dig.its
        out.append(d, n);
        out += '.';
        out.append(d + n, k - n);
    } else if (kMin < n && n <= 0) {   // 0.000digits
        out += "0.";
        out.append((size_t)-n, '0');
        out.append(d, k);
    } else {   // d.igitse+XX
        out += d[0];
        if (k > 1) {
            out += '.';
            out.append(d + 1, k - 1);
        }
        int e = n - 1;
        out += 'e';
        out += e < 0 ? '-' : '+';
        if (e < 0) e = -e;
        char eb[4];
        int el = 0;
        if (e < 10) {
            eb[el++] = '0';
            eb[el++] = (char)('0' + e);
        } else if (e < 100) {
            eb[el++] = (char)('0' + e / 10);
            eb[el++] = (char)('0' + e % 10);
        } else {
            eb[el++] = (char)('0' + e / 100);
            eb[el++] = (char)('0' + (e / 10) % 10);
            eb[el++] = (char)('0' + e % 10);
        }
        out.append(eb, el);
    }
}

}  // namespace

void json_number(std::string& out, double v) { append_json_number(out, v); }

std::string format_spectrum_json(const double* b, size_t n, double f_start, double f_step, size_t source_n) {
    // spectra.cpp:161-176: an object with keys in sorted order, two-space indentation, one array element
    // per line, then the writer's newline
    std::string out = "{\n  \"f_start_hz\": ";
    append_json_number(out, f_start);
    out += ",\n  \"f_step_hz\": ";
    append_json_number(out, f_step);
    auto array = [&](const char* key, auto&& value) {
        out += ",\n  \"";
        out += key;
        out += "\": ";
        if (n == 0) {
            out += "[]";
            return;
        }
        out += "[\n";
        for (size_t k = 0; k < n; ++k) {
            out += "    ";
            append_json_number(out, value(k));
            out += k + 1 < n ? ",\n" : "\n";
        }
        out += "  ]";
    };
    array("im", [&](size_t k) { return b[2 * k + 1]; });
    array("magnitude_db", [&](size_t k) { return magnitude_db(b[2 * k], b[2 * k + 1]); });
    array("re", [&](size_t k) { return b[2 * k]; });
    out += ",\n  \"source_n\": " + std::to_string(source_n) + "\n}\n";
    return out;
}

void write_spectrum_json_file(const double* b, size_t n, double f_start, double f_step, size_t source_n,
                              const std::string& path) {
    write_text_file(format_spectrum_json(b, n, f_start, f_step, source_n), path, "cannot open spectrum file for writing: ",
                    "spectrum json");
}

HostTrace parse_trace_csv(const char* data, size_t len, const std::string& origin) {
    std::vector<double> times, values;
    size_t line_no = 0;
    bool first_content = true;
    size_t pos = 0;
    while (pos < len) {   // std::getline: every '\n'-terminated line, plus a non-empty tail
        const char* nl = static_cast<const char*>(memchr(data + pos, '\n', len - pos));
        const size_t end = nl ? (size_t)(nl - data) : len;
        std::string_view line(data + pos, end - pos);
        pos = end + 1;
        ++line_no;
        if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
        if (line.find_first_not_of(" \t") == std::string_view::npos) continue;
        double t = 0.0, x = 0.0;
        if (!parse_row(line, t, x)) {
            if (first_content) {   // optional header
                first_content = false;
                continue;
            }
            throw ParseError(origin + ": malformed row at line " + std::to_string(line_no), line_no);
        }
        first_content = false;
        times.push_back(t);
        values.push_back(x);
    }
    if (times.size() < 2) throw FormatError(origin + ": need at least 2 samples to infer the sample rate");
    std::vector<double> steps(times.size() - 1);
    for (size_t i = 0; i + 1 < times.size(); ++i) steps[i] = times[i + 1] - times[i];
    std::vector<double> sorted = steps;
    std::nth_element(sorted.begin(), sorted.begin() + sorted.size() / 2, sorted.end());
    const double median = sorted[sorted.size() / 2];
    if (!(median > 0.0)) throw FormatError(origin + ": time column is not strictly increasing");
    for (size_t i = 0; i < steps.size(); ++i)
        if (std::abs(steps[i] - median) > 1e-6 * median)
            throw FormatError(origin + ": non-uniform time step between rows " + std::to_string(i + 1) + " and " +
                              std::to_string(i + 2) + " (got " + std::to_string(steps[i]) + " s, expected " +
                              std::to_string(median) + " s)");
    HostTrace tr;
    tr.samples = std::move(values);
    tr.fs = 1.0 / median;
    tr.t0 = times.front();
    // validate_trace (types.cpp:20-27)
    if (!(tr.fs > 0.0) || !std::isfinite(tr.fs))
        throw std::invalid_argument("trace: sample rate must be positive and finite");
    for (double v : tr.samples)
        if (!std::isfinite(v)) throw std::invalid_argument("trace: non-finite sample");
    if (!std::isfinite(tr.t0)) throw std::invalid_argument("trace: non-finite start time");
    return tr;
}

HostSpectrum parse_spectrum_csv(const char* data, size_t len, const std::string& origin) {
    std::vector<double> freqs, bins;
    size_t line_no = 0, pos = 0;
    bool first_content = true;
    while (pos < len) {
        const char* nl = static_cast<const char*>(memchr(data + pos, '\n', len - pos));
        const size_t end = nl ? (size_t)(nl - data) : len;
        std::string_view line(data + pos, end - pos);
        pos = end + 1;
        ++line_no;
        if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
        if (line.find_first_not_of(" \t") == std::string_view::npos) continue;
        double vals[4];
        std::string_view rest = line;
        bool ok = true;
        for (int c = 0; c < 4 && ok; ++c) {   // spectra.cpp:106-121: exactly four fields
            const size_t comma = rest.find(',');
            std::string_view field = c < 3 ? rest.substr(0, comma) : rest;
            if (c < 3) {
                if (comma == std::string_view::npos) {
                    ok = false;
                    break;
                }
                rest = rest.substr(comma + 1);
            } else if (comma != std::string_view::npos) {
                ok = false;
                break;
            }
            ok = parse_double(field, vals[c]);
        }
        if (!ok) {
            if (first_content) {
                first_content = false;
                continue;
            }
            throw ParseError(origin + ": malformed row at line " + std::to_string(line_no), line_no);
        }
        first_content = false;
        freqs.push_back(vals[0]);
        bins.push_back(vals[1]);
        bins.push_back(vals[2]);
    }
    if (bins.empty()) throw FormatError(origin + ": no spectrum rows");
    HostSpectrum s;
    s.f_start = freqs.front();
    const size_t n = freqs.size();
    if (n == 1) {
        s.f_step = 0.0;
    } else {
        const double step = (freqs.back() - freqs.front()) / static_cast<double>(n - 1);
        if (!(step > 0.0)) throw FormatError(origin + ": frequency axis is not increasing");
        for (size_t k = 0; k + 1 < n; ++k)
            if (std::abs(freqs[k + 1] - freqs[k] - step) > 1e-6 * step)
                throw FormatError(origin + ": non-uniform frequency step near row " + std::to_string(k + 1));
        s.f_step = step;
    }
    s.bins = std::move(bins);
    s.source_n = n;
    return s;
}

HostSpectrum read_spectrum_csv_file(const std::string& path) {
    if (path == "-") {
        const std::string s = slurp(stdin);
        return parse_spectrum_csv(s.data(), s.size(), "stdin");
    }
    FILE* f = fopen(path.c_str(), "rb");
    if (!f) throw IoError("cannot open spectrum file: " + path);
    const std::string s = slurp(f);
    fclose(f);
    return parse_spectrum_csv(s.data(), s.size(), path);
}

void append_g17(std::string& out, double v) {
    char buf[64];
    char* p = put_g17(buf, buf + sizeof buf, v);
    out.append(buf, p - buf);
}

void write_text_file(const std::string& body, const std::string& path, const char* open_msg, const char* what) {
    FILE* f = stdout;
    if (path != "-") {
        f = fopen(path.c_str(), "wb");
        if (!f) throw IoError(std::string(open_msg) + path);
    }
    const bool ok = fwrite(body.data(), 1, body.size(), f) == body.size();
    finish_out(f, ok, what);
}

HostTrace read_trace_csv_file(const std::string& path) {
    if (path == "-") {
        const std::string s = slurp(stdin);
        return parse_trace_csv(s.data(), s.size(), "stdin");
    }
    FILE* f = fopen(path.c_str(), "rb");
    if (!f) throw IoError("cannot open trace file: " + path);
    const std::string s = slurp(f);
    fclose(f);
    return parse_trace_csv(s.data(), s.size(), path);
}

void write_trace_csv_file(const double* samples, size_t n, double fs, double t0, const std::string& path) {
    FILE* f = open_out(path, "trace");
    // validate_trace runs inside write_trace_csv, after the file was opened (signals.cpp:178-195)
    auto invalid = [&](const char* msg) {
        if (f != stdout) fclose(f);
        throw std::invalid_argument(msg);
    };
    if (n == 0) invalid("trace: no samples");
    if (!(fs > 0.0) || !std::isfinite(fs)) invalid("trace: sample rate must be positive and finite");
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(samples[i])) invalid("trace: non-finite sample");
    if (!std::isfinite(t0)) invalid("trace: non-finite start time");
    std::string out = "time_s,amplitude\n";
    out.reserve(out.size() + n * 50);
    const double dt = 1.0 / fs;
    char buf[96];
    for (size_t i = 0; i < n; ++i) {
        char* p = put_g17(buf, buf + sizeof buf, t0 + static_cast<double>(i) * dt);
        *p++ = ',';
        p = put_g17(p, buf + sizeof buf, samples[i]);
        *p++ = '\n';
        out.append(buf, p - buf);
    }
    const bool ok = fwrite(out.data(), 1, out.size(), f) == out.size();
    finish_out(f, ok, "trace csv");
}

std::string format_spectrum_csv(const double* b, size_t n, double f_start, double f_step) {
    std::string out = "frequency_hz,re,im,magnitude_db\n";
    out.reserve(out.size() + n * 100);
    char buf[160];
    for (size_t k = 0; k < n; ++k) {
        const double re = b[2 * k], im = b[2 * k + 1];
        char* e = buf + sizeof buf;
        char* p = put_g17(buf, e, f_start + static_cast<double>(k) * f_step);   // Spectrum::frequency
        *p++ = ',';
        p = put_g17(p, e, re);
        *p++ = ',';
        p = put_g17(p, e, im);
        *p++ = ',';
        p = put_g17(p, e, magnitude_db(re, im));
        *p++ = '\n';
        out.append(buf, p - buf);
    }
    return out;
}

void write_spectrum_csv_file(const double* b, size_t n, double f_start, double f_step, const std::string& path) {
    FILE* f = open_out(path, "spectrum");
    const std::string out = format_spectrum_csv(b, n, f_start, f_step);
    const bool ok = fwrite(out.data(), 1, out.size(), f) == out.size();
    finish_out(f, ok, "spectrum csv");
}

void parallel_for(size_t count, int threads, const std::function<void(size_t)>& fn) {
    if (count == 0) return;
    size_t nt = threads > 0 ? (size_t)threads : std::max(1u, std::thread::hardware_concurrency());
    nt = std::min(nt, count);
    std::vector<std::exception_ptr> err(count);
    std::atomic<size_t> next{0};
    auto work = [&] {
        for (size_t i; (i = next.fetch_add(1)) < count;) {
            try {
                fn(i);
            } catch (...) {
                err[i] = std::current_exception();
            }
        }
    };
    std::vector<std::thread> pool;
    for (size_t t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

}  // namespace skg
