// .tns tensor files and a binary sidecar (host side of the input path; include/cpfit_io.h).
//
// Restates the reference's text format and diagnostics (proj/core/src/io.cpp:15-19, 92-215,
// io.hpp:18-30):
//   tns <N> <I1> ... <IN> <nnz>            header (first line)
//   <i1> ... <iN> <value>                  nnz entry lines, 1-based indices
// values written with the shortest round-trip form (std::to_chars), numbers parsed with
// std::from_chars (no leading '+', whole token), blank-separated tokens, a trailing '\r'
// dropped, lines after the nnz-th ignored, and io_error messages "<name>:<line>: <what>" for
// the first offending line in file order.
//
// What changes is the speed: the reference parses line by line on one thread through
// istringstream tokenisers (a 10M-entry BASELINE config-4 file is minutes); here the file is read
// in one block, the body is cut into per-thread ranges at line boundaries, each thread counts its
// lines, and after a prefix sum every thread parses straight into the caller's arrays; writers
// format per-thread chunks that are written in order. A binary sidecar (<path>.cpfbin: header,
// AoS int64 coordinates, fp64 values, stamped with the text file's size and mtime) turns later
// reads into one sequential copy.
#include "../../include/cpfit_io.h"

#include <sys/stat.h>

#include <cstdint>

#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_ioerr;

struct io_error : std::runtime_error {
    explicit io_error(const std::string& w) : std::runtime_error(w) {}
};

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const io_error& e) {
        g_ioerr = e.what();
        return 4;
    } catch (const std::invalid_argument& e) {
        g_ioerr = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_ioerr = e.what();
        return 3;
    }
}

int io_threads() {
    const unsigned n = std::thread::hardware_concurrency();
    return (int)std::max(1u, std::min(n, 64u));
}

// run f(t) for t in [0, n) on n threads (the calling thread takes t = 0)
template <class F>
void parallel(int n, F&& f) {
    std::vector<std::thread> th;
    for (int t = 1; t < n; ++t) th.emplace_back([&, t] { f(t); });
    f(0);
    for (auto& x : th) x.join();
}

std::string read_file(const std::string& path) {
    FILE* fp = std::fopen(path.c_str(), "rb");
    if (!fp) throw io_error("cannot open '" + path + "' for reading");
    std::string s;
    std::fseek(fp, 0, SEEK_END);
    const long sz = std::ftell(fp);
    std::fseek(fp, 0, SEEK_SET);
    if (sz > 0) {
        s.resize((size_t)sz);
        const size_t got = std::fread(&s[0], 1, (size_t)sz, fp);
        s.resize(got);
    }
    std::fclose(fp);
    return s;
}

// one line [b, e) without its '\n' and trailing '\r'
struct Line {
    const char* b;
    const char* e;
};

bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

// whitespace tokens of a line (istringstream >> std::string semantics)
int split_ws(Line l, Line* tok, int cap) {
    int n = 0;
    const char* p = l.b;
    while (p < l.e) {
        while (p < l.e && is_ws(*p)) ++p;
        if (p >= l.e) break;
        const char* q = p;
        while (q < l.e && !is_ws(*q)) ++q;
        if (n < cap) tok[n] = Line{p, q};
        ++n;
        p = q;
    }
    return n;
}

std::string str(Line t) { return std::string(t.b, t.e); }

// a parse failure at a line (message as LineReader::fail, io.cpp:43-45)
struct Fail {
    long long line = -1;
    std::string what;
};

bool parse_int(Line t, long long& v) {
    auto r = std::from_chars(t.b, t.e, v);
    return r.ec == std::errc{} && r.ptr == t.e;
}
bool parse_double(Line t, double& v) {
    auto r = std::from_chars(t.b, t.e, v);
    return r.ec == std::errc{} && r.ptr == t.e;
}

struct Header {
    int order = 0;
    int64_t dims[8] = {};
    int64_t nnz = 0;
    size_t body = 0;  // offset of the first body line
};

// the first line (io.cpp:104-121)
Header parse_header(const std::string& text, const std::string& name) {
    Header h;
    if (text.empty()) throw io_error(name + ": unexpected end of file, expected tns header");
    const char* b = text.data();
    const char* nl = static_cast<const char*>(std::memchr(b, '\n', text.size()));
    const char* e = nl ? nl : b + text.size();
    h.body = nl ? (size_t)(nl - b) + 1 : text.size();
    if (e > b && e[-1] == '\r') --e;
    auto fail = [&](const std::string& w) { throw io_error(name + ":1: " + w); };
    Line tok[16];
    const int nt = split_ws(Line{b, e}, tok, 16);
    if (nt == 0 || str(tok[0]) != "tns") fail("expected 'tns' header");
    if (nt < 2) fail("tns header needs an order");
    long long order = 0;
    if (!parse_int(tok[1], order)) fail("expected an integer, got '" + str(tok[1]) + "'");
    if (order < 1) fail("tensor order must be >= 1");
    if ((long long)nt != order + 3) fail("tns header needs <N> mode sizes and a count");
    if (order > 8) throw std::invalid_argument("tns: this build supports tensor order <= 8");
    h.order = (int)order;
    for (int n = 0; n < h.order; ++n) {
        long long d = 0;
        if (!parse_int(tok[2 + n], d)) fail("expected an integer, got '" + str(tok[2 + n]) + "'");
        if (d < 1) fail("mode sizes must be >= 1");
        h.dims[n] = d;
    }
    long long nnz = 0;
    if (!parse_int(tok[nt - 1], nnz)) fail("expected an integer, got '" + str(tok[nt - 1]) + "'");
    if (nnz < 0) fail("entry count must be >= 0");
    h.nnz = nnz;
    return h;
}

// Entry lines (io.cpp:128-147), parsed by all threads: coords (0-based, AoS) and values.
void parse_body(const std::string& text, const Header& h, const std::string& name, int64_t* coords, double* values) {
    const int N = h.order;
    if (h.nnz == 0) return;
    const char* base = text.data();
    const size_t lo = h.body, hi = text.size();
    const int T = (int)std::max<int64_t>(1, std::min<int64_t>(io_threads(), (int64_t)((hi - lo) >> 16) + 1));
    // thread ranges cut at line starts
    std::vector<size_t> cut((size_t)T + 1, hi);
    cut[0] = lo;
    for (int t = 1; t < T; ++t) {
        size_t p = lo + (hi - lo) * (size_t)t / (size_t)T;
        p = std::max(p, cut[(size_t)t - 1]);
        const void* nl = p < hi ? std::memchr(base + p, '\n', hi - p) : nullptr;
        cut[(size_t)t] = nl ? (size_t)(static_cast<const char*>(nl) - base) + 1 : hi;
    }
    // lines per range (a last line without '\n' still counts, io.cpp getline)
    std::vector<int64_t> cnt((size_t)T, 0);
    parallel(T, [&](int t) {
        const char* p = base + cut[(size_t)t];
        const char* e = base + cut[(size_t)t + 1];
        int64_t c = 0;
        while (p < e) {
            const void* nl = std::memchr(p, '\n', (size_t)(e - p));
            ++c;
            p = nl ? static_cast<const char*>(nl) + 1 : e;
        }
        cnt[(size_t)t] = c;
    });
    std::vector<int64_t> first((size_t)T + 1, 0);
    for (int t = 0; t < T; ++t) first[(size_t)t + 1] = first[(size_t)t] + cnt[(size_t)t];
    // a truncated body is reported only after the lines that exist parsed cleanly (the
    // reference reads line by line, so an earlier bad line wins)
    std::vector<Fail> fails((size_t)T);
    const std::string nline = std::to_string(N);
    parallel(T, [&](int t) {
        const char* p = base + cut[(size_t)t];
        const char* e = base + cut[(size_t)t + 1];
        int64_t k = first[(size_t)t];  // entry index of the next line
        Line tok[10];
        while (p < e && k < h.nnz) {
            const void* nlp = std::memchr(p, '\n', (size_t)(e - p));
            const char* le = nlp ? static_cast<const char*>(nlp) : e;
            Line l{p, le};
            if (l.e > l.b && l.e[-1] == '\r') --l.e;
            p = nlp ? le + 1 : e;
            const long long lineno = 2 + k;  // header is line 1
            auto fail = [&](const std::string& w) {
                fails[(size_t)t] = Fail{lineno, name + ":" + std::to_string(lineno) + ": " + w};
            };
            const int nt = split_ws(l, tok, 10);
            if (nt != N + 1) {
                fail("entry needs " + nline + " indices and a value");
                return;
            }
            for (int n = 0; n < N; ++n) {
                long long c = 0;
                if (!parse_int(tok[n], c)) {
                    fail("expected an integer, got '" + str(tok[n]) + "'");
                    return;
                }
                if (c < 1 || c > h.dims[n]) {
                    fail("index out of bounds");
                    return;
                }
                if (coords) coords[k * N + n] = c - 1;
            }
            double v = 0.0;
            if (!parse_double(tok[N], v)) {
                fail("expected a number, got '" + str(tok[N]) + "'");
                return;
            }
            if (values) values[k] = v;
            ++k;
        }
    });
    for (const Fail& f : fails)
        if (f.line >= 0) throw io_error(f.what);  // ranges are in file order: the first is the earliest
    if (first[(size_t)T] < h.nnz) throw io_error(name + ": unexpected end of file, expected tensor entry");
}

// ---- binary sidecar ---------------------------------------------------------------------
constexpr char kMagic[8] = {'C', 'P', 'F', 'I', 'T', 'T', 'N', 'S'};
struct SideHead {
    char magic[8];
    uint32_t version, order;
    uint64_t src_size;
    int64_t src_mtime_ns;
    int64_t nnz;
    int64_t dims[8];
};

bool stat_of(const std::string& path, uint64_t& size, int64_t& mtime_ns) {
    struct stat st {};
    if (::stat(path.c_str(), &st) != 0) return false;
    size = (uint64_t)st.st_size;
    mtime_ns = (int64_t)st.st_mtim.tv_sec * 1000000000LL + st.st_mtim.tv_nsec;
    return true;
}

std::string sidecar_path(const std::string& path) { return path + ".cpfbin"; }

// header of a sidecar that still matches its text file (size and mtime), else false
bool sidecar_head(const std::string& path, SideHead& sh) {
    uint64_t sz = 0;
    int64_t mt = 0;
    if (!stat_of(path, sz, mt)) return false;
    FILE* fp = std::fopen(sidecar_path(path).c_str(), "rb");
    if (!fp) return false;
    const bool ok = std::fread(&sh, sizeof(sh), 1, fp) == 1 && std::memcmp(sh.magic, kMagic, 8) == 0 &&
                    sh.version == 1 && sh.order >= 1 && sh.order <= 8 && sh.src_size == sz &&
                    sh.src_mtime_ns == mt && sh.nnz >= 0;
    std::fclose(fp);
    return ok;
}

void sidecar_body(const std::string& path, const SideHead& sh, int64_t* coords, double* values) {
    FILE* fp = std::fopen(sidecar_path(path).c_str(), "rb");
    if (!fp) throw io_error("cannot open '" + sidecar_path(path) + "' for reading");
    std::fseek(fp, (long)sizeof(SideHead), SEEK_SET);
    const size_t nc = (size_t)sh.nnz * sh.order;
    bool ok = true;
    if (coords)
        ok = std::fread(coords, sizeof(int64_t), nc, fp) == nc;
    else
        std::fseek(fp, (long)(sizeof(int64_t) * nc), SEEK_CUR);
    if (ok && values) ok = std::fread(values, sizeof(double), (size_t)sh.nnz, fp) == (size_t)sh.nnz;
    std::fclose(fp);
    if (!ok) throw io_error(sidecar_path(path) + ": truncated sidecar");
}

void write_sidecar(const std::string& path, const Header& h, const int64_t* coords, const double* values) {
    SideHead sh{};
    std::memcpy(sh.magic, kMagic, 8);
    sh.version = 1;
    sh.order = (uint32_t)h.order;
    if (!stat_of(path, sh.src_size, sh.src_mtime_ns)) return;
    sh.nnz = h.nnz;
    for (int n = 0; n < h.order; ++n) sh.dims[n] = h.dims[n];
    const std::string tmp = sidecar_path(path) + ".tmp";
    FILE* fp = std::fopen(tmp.c_str(), "wb");
    if (!fp) return;  // a read-only directory just means no sidecar
    bool ok = std::fwrite(&sh, sizeof(sh), 1, fp) == 1;
    const size_t nc = (size_t)h.nnz * h.order;
    ok = ok && std::fwrite(coords, sizeof(int64_t), nc, fp) == nc;
    ok = ok && std::fwrite(values, sizeof(double), (size_t)h.nnz, fp) == (size_t)h.nnz;
    ok = (std::fclose(fp) == 0) && ok;
    if (ok)
        std::rename(tmp.c_str(), sidecar_path(path).c_str());
    else
        std::remove(tmp.c_str());
}

// ---- writers ------------------------------------------------------------------------------
// format_double (io.cpp:15-19): shortest round-trip digits
inline char* fmt_double(char* p, double x) { return std::to_chars(p, p + 32, x).ptr; }
inline char* fmt_int(char* p, long long x) { return std::to_chars(p, p + 24, x).ptr; }

void write_header(std::string& s, int order, const int64_t* dims, int64_t nnz) {
    s += "tns " + std::to_string(order);
    for (int n = 0; n < order; ++n) s += ' ' + std::to_string(dims[n]);
    s += ' ' + std::to_string(nnz) + '\n';
}

// entries [0, count) formatted by `line(k, p) -> end` on all threads, written in order
template <class L>
void write_entries(const std::string& path, const std::string& head, int64_t count, size_t max_line, L&& line) {
    FILE* fp = std::fopen(path.c_str(), "wb");
    if (!fp) throw io_error("cannot open '" + path + "' for writing");
    bool ok = std::fwrite(head.data(), 1, head.size(), fp) == head.size();
    const int64_t chunk = 1 << 18;
    const int T = io_threads();
    std::vector<std::string> buf((size_t)T);
    for (int64_t k0 = 0; ok && k0 < count; k0 += chunk * T) {
        parallel(T, [&](int t) {
            const int64_t a = k0 + chunk * t, b = std::min(count, a + chunk);
            std::string& s = buf[(size_t)t];
            s.clear();
            if (a >= b) return;
            s.resize((size_t)(b - a) * max_line);
            char* p = &s[0];
            for (int64_t k = a; k < b; ++k) p = line(k, p);
            s.resize((size_t)(p - s.data()));
        });
        for (int t = 0; t < T && ok; ++t) ok = std::fwrite(buf[(size_t)t].data(), 1, buf[(size_t)t].size(), fp) == buf[(size_t)t].size();
    }
    ok = (std::fclose(fp) == 0) && ok;
    if (!ok) throw io_error("cannot write '" + path + "'");
}

void check_shape(int order, const int64_t* dims) {
    if (order < 1 || order > 8) throw std::invalid_argument("tns: order must be in [1, 8]");
    for (int n = 0; n < order; ++n)
        if (dims[n] < 1) throw std::invalid_argument("Shape: every mode size must be >= 1");
}

}  // namespace

extern "C" {

const char* cpfit_io_last_error(void) { return g_ioerr.c_str(); }

int cpfit_format_double(double x, char* buf, int cap) {
    return guard([&] {
        char tmp[40];
        char* e = fmt_double(tmp, x);
        const int n = (int)(e - tmp);
        if (cap < n + 1) throw std::invalid_argument("format_double: buffer too small");
        std::memcpy(buf, tmp, (size_t)n);
        buf[n] = '\0';
    });
}

int cpfit_tns_read(const char* path, int sidecar, int* order, int64_t* dims, int64_t* nnz, int64_t* coords,
                   double* values, int64_t cap, int* from_sidecar) {
    return guard([&] {
        const std::string p(path);
        if (from_sidecar) *from_sidecar = 0;
        SideHead sh{};
        if (sidecar && sidecar_head(p, sh)) {
            *order = (int)sh.order;
            for (int n = 0; n < (int)sh.order; ++n) dims[n] = sh.dims[n];
            *nnz = sh.nnz;
            if (coords || values) {
                if (cap < sh.nnz) throw std::invalid_argument("tns: output capacity below the entry count");
                sidecar_body(p, sh, coords, values);
            }
            if (from_sidecar) *from_sidecar = 1;
            return;
        }
        const std::string text = read_file(p);
        const Header h = parse_header(text, p);
        *order = h.order;
        for (int n = 0; n < h.order; ++n) dims[n] = h.dims[n];
        *nnz = h.nnz;
        if (!coords && !values && sidecar != 2) return;
        if ((coords || values) && cap < h.nnz) throw std::invalid_argument("tns: output capacity below the entry count");
        if (sidecar == 2 && !(coords && values)) {
            std::vector<int64_t> c((size_t)h.nnz * h.order);
            std::vector<double> v((size_t)h.nnz);
            parse_body(text, h, p, c.data(), v.data());
            write_sidecar(p, h, c.data(), v.data());
            if (coords) std::memcpy(coords, c.data(), sizeof(int64_t) * c.size());
            if (values) std::memcpy(values, v.data(), sizeof(double) * v.size());
            return;
        }
        parse_body(text, h, p, coords, values);
        if (sidecar == 2) write_sidecar(p, h, coords, values);
    });
}

int cpfit_tns_read_dense(const char* path, int sidecar, int* order, int64_t* dims, int64_t* K, double* values,
                         int64_t cap) {
    return guard([&] {
        int64_t nnz = 0;
        int o = 0;
        int64_t d[8];
        if (int rc = cpfit_tns_read(path, sidecar, &o, d, &nnz, nullptr, nullptr, 0, nullptr)) {
            if (rc == 4) throw io_error(g_ioerr);
            if (rc == 1) throw std::invalid_argument(g_ioerr);
            throw std::runtime_error(g_ioerr);
        }
        int64_t k = 1;
        for (int n = 0; n < o; ++n) {
            if (k > INT64_MAX / d[n]) throw std::invalid_argument("Shape: element count overflows the index range");
            k *= d[n];
        }
        *order = o;
        for (int n = 0; n < o; ++n) dims[n] = d[n];
        *K = k;
        if (!values) return;
        if (cap < k) throw std::invalid_argument("tns: output capacity below the element count");
        std::vector<int64_t> c((size_t)nnz * o);
        std::vector<double> v((size_t)nnz);
        if (int rc = cpfit_tns_read(path, sidecar, &o, d, &nnz, c.data(), v.data(), nnz, nullptr)) {
            if (rc == 4) throw io_error(g_ioerr);
            if (rc == 1) throw std::invalid_argument(g_ioerr);
            throw std::runtime_error(g_ioerr);
        }
        std::fill(values, values + k, 0.0);
        // io.cpp:196-200: values[offset] = value in file order (a later duplicate wins)
        for (int64_t i = 0; i < nnz; ++i) {
            int64_t off = 0, stride = 1;
            for (int n = 0; n < o; ++n) {
                off += c[(size_t)(i * o + n)] * stride;
                stride *= d[n];
            }
            values[off] = v[(size_t)i];
        }
    });
}

int cpfit_tns_write(const char* path, int order, const int64_t* dims, int64_t nnz, const int64_t* coords,
                    const double* values) {
    return guard([&] {
        check_shape(order, dims);
        if (nnz < 0) throw std::invalid_argument("tns: nnz must be >= 0");
        std::string head;
        write_header(head, order, dims, nnz);
        // io.cpp:151-159: "c+1 " per mode, then the value
        write_entries(path, head, nnz, (size_t)order * 21 + 32, [&](int64_t k, char* p) {
            for (int n = 0; n < order; ++n) {
                p = fmt_int(p, coords[k * order + n] + 1);
                *p++ = ' ';
            }
            p = fmt_double(p, values[k]);
            *p++ = '\n';
            return p;
        });
    });
}

int cpfit_tns_write_dense(const char* path, int order, const int64_t* dims, const double* values) {
    return guard([&] {
        check_shape(order, dims);
        int64_t K = 1;
        for (int n = 0; n < order; ++n) K *= dims[n];
        std::string head;
        write_header(head, order, dims, K);
        // io.cpp:161-174: every element, first mode fastest
        write_entries(path, head, K, (size_t)order * 21 + 32, [&](int64_t flat, char* p) {
            int64_t rem = flat;
            for (int n = 0; n < order; ++n) {
                p = fmt_int(p, rem % dims[n] + 1);
                rem /= dims[n];
                *p++ = ' ';
            }
            p = fmt_double(p, values[flat]);
            *p++ = '\n';
            return p;
        });
    });
}

}  // extern "C"
