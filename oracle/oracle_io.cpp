// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp). Sequential restatement of the reference's
// .tns reader/writer (proj/core/src/io.cpp:15-19 format_double, :33-90 line reader and number
// parsing, :92-147 header/body, :151-205 read/write): getline-style lines with a trailing '\r'
// dropped, whitespace tokens as istringstream >> std::string splits them (classic-locale
// isspace), std::from_chars numbers, io_error "<name>:<line>: <what>". (stdio instead of
// iostreams: this library is loaded into Python with a statically linked libstdc++.)
// The product's multi-threaded parser/writer (paper_1105_5331_b200/csrc/io.cpp) is checked
// against these bytes, values and messages.
#include <cctype>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

struct io_error : std::runtime_error {
    explicit io_error(const std::string& w) : std::runtime_error(w) {}
};

struct Reader {
    FILE* is;
    std::string name;
    long line = 0;
    bool next(std::string& s) {  // std::getline: false only when nothing is left
        s.clear();
        int c = std::fgetc(is);
        if (c == EOF) return false;
        while (c != EOF && c != '\n') {
            s.push_back((char)c);
            c = std::fgetc(is);
        }
        ++line;
        if (!s.empty() && s.back() == '\r') s.pop_back();
        return true;
    }
    [[noreturn]] void fail(const std::string& w) const { throw io_error(name + ":" + std::to_string(line) + ": " + w); }
    std::string need(const std::string& what) {
        std::string s;
        if (!next(s)) throw io_error(name + ": unexpected end of file, expected " + what);
        return s;
    }
};

std::vector<std::string> tokens(const std::string& s) {
    std::vector<std::string> t;
    size_t i = 0;
    while (i < s.size()) {
        while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
        size_t j = i;
        while (j < s.size() && !std::isspace((unsigned char)s[j])) ++j;
        if (j > i) t.push_back(s.substr(i, j - i));
        i = j;
    }
    return t;
}

long long to_int(const std::string& t, const Reader& r) {
    long long v = 0;
    auto [p, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
    if (ec != std::errc{} || p != t.data() + t.size()) r.fail("expected an integer, got '" + t + "'");
    return v;
}

double to_double(const std::string& t, const Reader& r) {
    double v = 0;
    auto [p, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
    if (ec != std::errc{} || p != t.data() + t.size()) r.fail("expected a number, got '" + t + "'");
    return v;
}

std::string fmt(double x) {
    char b[64];
    auto [e, ec] = std::to_chars(b, b + sizeof b, x);
    return std::string(b, e);
}

}  // namespace

extern "C" {

const char* oracle_io_last_error() { return g_err.c_str(); }

// read_tns_file: header into order/dims/nnz; entries (0-based AoS coords, values) when non-null
int oracle_tns_read(const char* path, int* order, int64_t* dims, int64_t* nnz, int64_t* coords, double* values) {
    try {
        FILE* f = std::fopen(path, "rb");
        if (!f) throw io_error(std::string("cannot open '") + path + "' for reading");
        struct Closer {
            FILE* f;
            ~Closer() { std::fclose(f); }
        } closer{f};
        Reader r{f, path};
        const auto h = tokens(r.need("tns header"));
        if (h.empty() || h[0] != "tns") r.fail("expected 'tns' header");
        if (h.size() < 2) r.fail("tns header needs an order");
        const long long n = to_int(h[1], r);
        if (n < 1) r.fail("tensor order must be >= 1");
        if ((long long)h.size() != n + 3) r.fail("tns header needs <N> mode sizes and a count");
        for (long long m = 0; m < n; ++m) {
            const long long d = to_int(h[(size_t)(2 + m)], r);
            if (d < 1) r.fail("mode sizes must be >= 1");
            dims[m] = d;
        }
        const long long cnt = to_int(h.back(), r);
        if (cnt < 0) r.fail("entry count must be >= 0");
        *order = (int)n;
        *nnz = cnt;
        if (!coords && !values) return 0;
        for (long long i = 0; i < cnt; ++i) {
            const auto t = tokens(r.need("tensor entry"));
            if ((long long)t.size() != n + 1) r.fail("entry needs " + std::to_string(n) + " indices and a value");
            for (long long m = 0; m < n; ++m) {
                const long long c = to_int(t[(size_t)m], r);
                if (c < 1 || c > dims[m]) r.fail("index out of bounds");
                coords[i * n + m] = c - 1;
            }
            values[i] = to_double(t.back(), r);
        }
        return 0;
    } catch (const io_error& e) {
        g_err = e.what();
        return 4;
    }
}

// write_tns_file(SparseTensor)
int oracle_tns_write(const char* path, int order, const int64_t* dims, int64_t nnz, const int64_t* coords,
                     const double* values) {
    FILE* os = std::fopen(path, "wb");
    if (!os) {
        g_err = std::string("cannot open '") + path + "' for writing";
        return 4;
    }
    std::fprintf(os, "tns %d", order);
    for (int n = 0; n < order; ++n) std::fprintf(os, " %lld", (long long)dims[n]);
    std::fprintf(os, " %lld\n", (long long)nnz);
    for (int64_t i = 0; i < nnz; ++i) {
        for (int n = 0; n < order; ++n) std::fprintf(os, "%lld ", (long long)(coords[i * order + n] + 1));
        std::fprintf(os, "%s\n", fmt(values[i]).c_str());
    }
    std::fclose(os);
    return 0;
}

}  // extern "C"
