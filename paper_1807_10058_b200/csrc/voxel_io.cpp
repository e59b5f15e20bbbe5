// Voxel grids, spectrum CSV interchange and geometry exports (voxel_io.hpp).
//
// Formats follow the reference byte for byte where it writes text through
// printf-style formatting (%.17g CSV: voxel_io.cpp:238-261, spectral.cpp:180-188).
// Grid JSON is written compactly with sorted keys, integral doubles as "1.0"
// and the shortest round-trip digits otherwise — the layout nlohmann::json's
// dump() produces (voxel_io.cpp:84-95) — and parsed by a small strict JSON
// reader; the values round-trip exactly either way.
#include "voxel_io.hpp"

#include <algorithm>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <memory>
#include <set>
#include <sstream>
#include <thread>

namespace fcct::io {
namespace {

constexpr char kSpectrumColumns[] = "i,j,k,x,y,z,re,im,magnitude";

[[noreturn]] void malformed(const std::string& m) { throw FcctError(ST_MALFORMED, m); }
[[noreturn]] void io_failure(const std::string& m) { throw FcctError(ST_IO, m); }


// std::stod / std::stoi semantics: leading whitespace and a sign accepted,
// trailing characters left for the caller, failure on no conversion or range.
bool stod_like(const std::string& s, double& v, size_t* used = nullptr) {
    const char* b = s.c_str();
    char* e = nullptr;
    errno = 0;
    v = std::strtod(b, &e);
    if (e == b || errno == ERANGE) return false;
    if (used) *used = static_cast<size_t>(e - b);
    return true;
}

bool stoi_like(const std::string& s, int& v) {
    const char* b = s.c_str();
    char* e = nullptr;
    errno = 0;
    const long x = std::strtol(b, &e, 10);
    if (e == b || errno == ERANGE || x < INT32_MIN || x > INT32_MAX) return false;
    v = static_cast<int>(x);
    return true;
}

std::string read_file(const std::string& path, const std::string& what) {
    std::ifstream in(path, std::ios::binary);
    if (!in) io_failure("cannot open " + what + " " + path);
    std::ostringstream ss;
    ss << in.rdbuf();
    return ss.str();
}

int hw_threads() {
    const unsigned h = std::thread::hardware_concurrency();
    return static_cast<int>(h == 0 ? 1 : std::min(h, 64u));
}

// Runs f(begin, end) over [0, count) in contiguous chunks on a few threads.
template <typename F>
void parallel_chunks(int64_t count, int64_t min_chunk, F&& f) {
    const int64_t want = std::max<int64_t>(1, std::min<int64_t>(hw_threads(), count / std::max<int64_t>(1, min_chunk)));
    if (want <= 1) {
        f(0, count, 0);
        return;
    }
    std::vector<std::thread> pool;
    const int64_t per = (count + want - 1) / want;
    for (int64_t t = 0; t < want; ++t) {
        const int64_t b = t * per, e = std::min(count, b + per);
        if (b >= e) break;
        pool.emplace_back([&f, b, e, t] { f(b, e, static_cast<int>(t)); });
    }
    for (auto& th : pool) th.join();
}

// ---------------------------------------------------------------------------
// Minimal JSON (RFC 8259) reader: enough for grid documents and sidecars.
// ---------------------------------------------------------------------------
struct JVal {
    enum Kind { Null, Bool, Int, Float, Str, Arr, Obj } kind = Null;
    bool b = false;
    int64_t i = 0;
    double d = 0.0;
    std::string s;
    std::vector<JVal> arr;
    std::map<std::string, JVal> obj;
    bool is_number() const { return kind == Int || kind == Float; }
    double num() const { return kind == Int ? static_cast<double>(i) : d; }
};

struct JParser {
    const char* p;
    const char* end;
    explicit JParser(const std::string& text) : p(text.data()), end(text.data() + text.size()) {}

    [[noreturn]] void fail(const std::string& why) { throw std::runtime_error(why); }
    void ws() {
        while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
    }
    bool lit(const char* w) {
        const size_t L = std::strlen(w);
        if (static_cast<size_t>(end - p) >= L && std::memcmp(p, w, L) == 0) {
            p += L;
            return true;
        }
        return false;
    }
    static void put_utf8(std::string& o, uint32_t cp) {
        if (cp < 0x80) {
            o += static_cast<char>(cp);
        } else if (cp < 0x800) {
            o += static_cast<char>(0xC0 | (cp >> 6));
            o += static_cast<char>(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            o += static_cast<char>(0xE0 | (cp >> 12));
            o += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            o += static_cast<char>(0x80 | (cp & 0x3F));
        } else {
            o += static_cast<char>(0xF0 | (cp >> 18));
            o += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
            o += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            o += static_cast<char>(0x80 | (cp & 0x3F));
        }
    }
    uint32_t hex4() {
        if (end - p < 4) fail("truncated \\u escape");
        uint32_t v = 0;
        for (int k = 0; k < 4; ++k) {
            const char c = *p++;
            v <<= 4;
            if (c >= '0' && c <= '9') v |= static_cast<uint32_t>(c - '0');
            else if (c >= 'a' && c <= 'f') v |= static_cast<uint32_t>(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F') v |= static_cast<uint32_t>(c - 'A' + 10);
            else fail("bad \\u escape");
        }
        return v;
    }
    std::string str() {
        if (p >= end || *p != '"') fail("expected a string");
        ++p;
        std::string o;
        while (true) {
            if (p >= end) fail("unterminated string");
            const char c = *p++;
            if (c == '"') break;
            if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
            if (c != '\\') {
                o += c;
                continue;
            }
            if (p >= end) fail("unterminated escape");
            const char e = *p++;
            switch (e) {
                case '"': o += '"'; break;
                case '\\': o += '\\'; break;
                case '/': o += '/'; break;
                case 'b': o += '\b'; break;
                case 'f': o += '\f'; break;
                case 'n': o += '\n'; break;
                case 'r': o += '\r'; break;
                case 't': o += '\t'; break;
                case 'u': {
                    uint32_t cp = hex4();
                    if (cp >= 0xD800 && cp <= 0xDBFF) {
                        if (!lit("\\u")) fail("unpaired surrogate");
                        const uint32_t lo = hex4();
                        if (lo < 0xDC00 || lo > 0xDFFF) fail("unpaired surrogate");
                        cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                    } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
                        fail("unpaired surrogate");
                    }
                    put_utf8(o, cp);
                    break;
                }
                default: fail("bad escape");
            }
        }
        return o;
    }
    JVal number() {
        const char* b = p;
        bool integral = true;
        if (p < end && *p == '-') ++p;
        if (p >= end || !(*p >= '0' && *p <= '9')) fail("bad number");
        if (*p == '0') {
            ++p;
        } else {
            while (p < end && *p >= '0' && *p <= '9') ++p;
        }
        if (p < end && *p == '.') {
            integral = false;
            ++p;
            if (p >= end || !(*p >= '0' && *p <= '9')) fail("bad number");
            while (p < end && *p >= '0' && *p <= '9') ++p;
        }
        if (p < end && (*p == 'e' || *p == 'E')) {
            integral = false;
            ++p;
            if (p < end && (*p == '+' || *p == '-')) ++p;
            if (p >= end || !(*p >= '0' && *p <= '9')) fail("bad number");
            while (p < end && *p >= '0' && *p <= '9') ++p;
        }
        JVal v;
        const std::string tok(b, p);
        if (integral) {
            int64_t x = 0;
            const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), x);
            if (r.ec == std::errc()) {
                v.kind = JVal::Int;
                v.i = x;
                return v;
            }
        }
        v.kind = JVal::Float;
        v.d = std::strtod(tok.c_str(), nullptr);
        return v;
    }
    JVal value(int depth = 0) {
        if (depth > 256) fail("nesting too deep");
        ws();
        if (p >= end) fail("unexpected end of input");
        JVal v;
        const char c = *p;
        if (c == '{') {
            ++p;
            v.kind = JVal::Obj;
            ws();
            if (p < end && *p == '}') {
                ++p;
                return v;
            }
            while (true) {
                ws();
                std::string k = str();
                ws();
                if (p >= end || *p != ':') fail("expected ':'");
                ++p;
                v.obj[k] = value(depth + 1);
                ws();
                if (p < end && *p == ',') {
                    ++p;
                    continue;
                }
                if (p < end && *p == '}') {
                    ++p;
                    break;
                }
                fail("expected ',' or '}'");
            }
        } else if (c == '[') {
            ++p;
            v.kind = JVal::Arr;
            ws();
            if (p < end && *p == ']') {
                ++p;
                return v;
            }
            while (true) {
                v.arr.push_back(value(depth + 1));
                ws();
                if (p < end && *p == ',') {
                    ++p;
                    continue;
                }
                if (p < end && *p == ']') {
                    ++p;
                    break;
                }
                fail("expected ',' or ']'");
            }
        } else if (c == '"') {
            v.kind = JVal::Str;
            v.s = str();
        } else if (lit("true")) {
            v.kind = JVal::Bool;
            v.b = true;
        } else if (lit("false")) {
            v.kind = JVal::Bool;
        } else if (lit("null")) {
            v.kind = JVal::Null;
        } else {
            v = number();
        }
        return v;
    }
    JVal document() {
        JVal v = value();
        ws();
        if (p != end) fail("trailing characters after the JSON value");
        return v;
    }
};

JVal parse_json(const std::string& text, const std::string& what) {
    try {
        return JParser(text).document();
    } catch (const std::runtime_error& e) {
        malformed(what + " is not valid JSON: " + e.what());
    }
}

void json_escape(std::string& o, const std::string& s) {
    o += '"';
    for (const unsigned char c : s) {
        switch (c) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\b': o += "\\b"; break;
            case '\f': o += "\\f"; break;
            case '\n': o += "\\n"; break;
            case '\r': o += "\\r"; break;
            case '\t': o += "\\t"; break;
            default:
                if (c < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof(buf), "\\u%04x", c);
                    o += buf;
                } else {
                    o += static_cast<char>(c);
                }
        }
    }
    o += '"';
}

// Shortest round-trip digits laid out the way nlohmann::json dumps a double:
// fixed notation for decimal exponents in (-4, 15], ".0" on integral values,
// otherwise d.ddde+XX with at least two exponent digits; non-finite -> null.
void json_double(std::string& o, double v) {
    if (!std::isfinite(v)) {
        o += "null";
        return;
    }
    if (v == 0.0) {
        o += std::signbit(v) ? "-0.0" : "0.0";
        return;
    }
    char sci[64];
    const auto r = std::to_chars(sci, sci + sizeof(sci), v, std::chars_format::scientific);
    std::string t(sci, r.ptr);
    std::string sign;
    if (t[0] == '-') {
        sign = "-";
        t.erase(0, 1);
    }
    const size_t epos = t.find('e');
    const int e10 = std::atoi(t.c_str() + epos + 1);
    std::string digits;
    for (size_t k = 0; k < epos; ++k)
        if (t[k] != '.') digits += t[k];
    const int len = static_cast<int>(digits.size());
    const int nexp = e10 + 1;  // position of the decimal point relative to the digits
    std::string out;
    if (len <= nexp && nexp <= 15) {
        out = digits + std::string(static_cast<size_t>(nexp - len), '0') + ".0";
    } else if (0 < nexp && nexp <= 15) {
        out = digits.substr(0, static_cast<size_t>(nexp)) + "." + digits.substr(static_cast<size_t>(nexp));
    } else if (-4 < nexp && nexp <= 0) {
        out = "0." + std::string(static_cast<size_t>(-nexp), '0') + digits;
    } else {
        out = digits.substr(0, 1);
        if (len > 1) out += "." + digits.substr(1);
        const int ex = nexp - 1;
        char eb[16];
        std::snprintf(eb, sizeof(eb), "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
        out += eb;
    }
    o += sign + out;
}

int read_grid_n(const JVal& doc) {  // voxel_io.cpp:41-49
    if (doc.kind != JVal::Obj) malformed("grid header lacks an integer n");
    const auto it = doc.obj.find("n");
    if (it == doc.obj.end() || it->second.kind != JVal::Int) malformed("grid header lacks an integer n");
    const int64_t n = it->second.i;
    if (n < 1 || n > 4096) malformed("grid size " + std::to_string(n) + " is out of range");
    return static_cast<int>(n);
}

std::map<std::string, std::string> read_metadata(const JVal& doc) {  // voxel_io.cpp:28-39
    std::map<std::string, std::string> out;
    const auto it = doc.obj.find("metadata");
    if (it == doc.obj.end() || it->second.kind == JVal::Null) return out;
    if (it->second.kind != JVal::Obj) malformed("grid metadata must be an object of strings");
    for (const auto& [k, v] : it->second.obj) {
        if (v.kind != JVal::Str) malformed("grid metadata must be an object of strings");
        out[k] = v.s;
    }
    return out;
}

void check_grid(const Grid& g) {  // check_grid_sizes (voxel_io.cpp:148-154)
    if (g.n < 1) throw FcctError(ST_SIZE_MISMATCH, "grid size must be >= 1");
    if (static_cast<int64_t>(g.values.size()) != cube(g.n))
        throw FcctError(ST_SIZE_MISMATCH, "grid carries " + std::to_string(g.values.size()) +
                                              " values for n=" + std::to_string(g.n));
}

void write_file(const std::string& path, const std::string& data, const std::string& what) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) io_failure("cannot write " + what + " " + path);
    out.write(data.data(), static_cast<std::streamsize>(data.size()));
    if (!out) io_failure("failed while writing " + path);
}

// real_coords (chebyshev.cpp:87-97) of one node's (x, y, z).
std::array<double, 3> real_coords(const std::array<std::complex<double>, 3>& s) {
    const std::complex<double> xt = 0.5 * (s[0] + s[2]);
    const std::complex<double> zt = (s[0] - s[2]) / std::complex<double>{0.0, 2.0};
    const double residue = std::max({std::abs(xt.imag()), std::abs(s[1].imag()), std::abs(zt.imag())});
    if (residue > 1e-8)
        throw FcctError(ST_INVALID_ARGUMENT, "real_coords: imaginary residue " + std::to_string(residue) +
                                                 " exceeds 1e-8; point is not the image of a torus point");
    return {xt.real(), s[1].real(), zt.real()};
}

}  // namespace

// ---------------------------------------------------------------------------
double parse_param(const std::string& text) {
    const auto bad = [&] { throw FcctError(ST_INVALID_ARGUMENT, "cannot parse grid offset '" + text + "'"); };
    if (text.empty()) throw FcctError(ST_INVALID_ARGUMENT, "empty grid offset");
    const auto slash = text.find('/');
    if (slash != std::string::npos) {
        double num = 0, den = 0;
        size_t used = 0, used_den = 0;
        const std::string num_text = text.substr(0, slash), den_text = text.substr(slash + 1);
        if (!stod_like(num_text, num, &used) || !stod_like(den_text, den, &used_den)) bad();
        if (used != slash || used_den != den_text.size() || den == 0.0) bad();
        return num / den;
    }
    double v = 0;
    size_t used = 0;
    if (!stod_like(text, v, &used) || used != text.size()) bad();
    return v;
}

Params parse_params(const std::string& text) {
    const auto first = text.find(',');
    const auto second = first == std::string::npos ? std::string::npos : text.find(',', first + 1);
    if (first == std::string::npos || second == std::string::npos || text.find(',', second + 1) != std::string::npos)
        throw FcctError(ST_INVALID_ARGUMENT, "grid offsets must be 'r,s,t', got '" + text + "'");
    return Params{parse_param(text.substr(0, first)), parse_param(text.substr(first + 1, second - first - 1)),
                  parse_param(text.substr(second + 1))};
}

std::string encode_params(const Params& p) {
    return encode_param(p.r) + "," + encode_param(p.s) + "," + encode_param(p.t);
}

bool is_json_path(const std::string& path) {  // format_for_path (voxel_io.cpp:156-158)
    const auto slash = path.find_last_of('/');
    const std::string base = slash == std::string::npos ? path : path.substr(slash + 1);
    const auto dot = base.find_last_of('.');
    // std::filesystem::path::extension: a leading dot alone ("."/".json") is not an extension
    if (dot == std::string::npos || dot == 0 || base == "..") return false;
    return base.substr(dot) == ".json";
}

std::string metadata_json(const std::map<std::string, std::string>& m) {
    std::string o = "{";
    bool first = true;
    for (const auto& [k, v] : m) {
        if (!first) o += ',';
        first = false;
        json_escape(o, k);
        o += ':';
        json_escape(o, v);
    }
    return o + "}";
}

std::map<std::string, std::string> parse_metadata_json(const std::string& text) {
    if (text.empty()) return {};
    JVal doc;
    try {
        doc = JParser(text).document();
    } catch (const std::runtime_error& e) {
        throw FcctError(ST_INVALID_ARGUMENT, std::string("metadata is not valid JSON: ") + e.what());
    }
    JVal wrap;
    wrap.kind = JVal::Obj;
    wrap.obj["metadata"] = doc;
    try {
        return read_metadata(wrap);
    } catch (const FcctError& e) {
        throw FcctError(ST_INVALID_ARGUMENT, e.what());
    }
}

Grid load_grid(const std::string& path) {
    Grid g;
    if (is_json_path(path)) {  // load_grid_json (voxel_io.cpp:56-82)
        const std::string text = read_file(path, "grid file");
        const JVal doc = parse_json(text, "grid file " + path);
        g.n = read_grid_n(doc);
        const auto it = doc.obj.find("values");
        if (it == doc.obj.end() || it->second.kind != JVal::Arr) malformed("grid file lacks a values array");
        const auto& vals = it->second.arr;
        if (static_cast<int64_t>(vals.size()) != cube(g.n))
            throw FcctError(ST_SIZE_MISMATCH_IO, "grid file promises n=" + std::to_string(g.n) + " but carries " +
                                                     std::to_string(vals.size()) + " values");
        g.values.reserve(vals.size());
        for (const auto& v : vals) {
            if (!v.is_number()) malformed("grid values must all be numbers");
            g.values.push_back(v.num());
        }
        g.metadata = read_metadata(doc);
    } else {  // load_grid_raw (voxel_io.cpp:97-129)
        const std::string side = path + ".json";
        std::ifstream sin(side, std::ios::binary);
        if (!sin) malformed("raw grid " + path + " lacks its sidecar " + side);
        std::ostringstream ss;
        ss << sin.rdbuf();
        const JVal doc = parse_json(ss.str(), "grid sidecar");
        g.n = read_grid_n(doc);
        g.metadata = read_metadata(doc);
        std::ifstream in(path, std::ios::binary | std::ios::ate);
        if (!in) io_failure("cannot open grid payload " + path);
        const int64_t bytes = static_cast<int64_t>(in.tellg());
        const int64_t expected = cube(g.n) * static_cast<int64_t>(sizeof(double));
        if (bytes != expected)
            throw FcctError(ST_SIZE_MISMATCH_IO, "raw grid payload is " + std::to_string(bytes) + " bytes, header n=" +
                                                     std::to_string(g.n) + " requires " + std::to_string(expected));
        in.seekg(0);
        g.values.resize(static_cast<size_t>(cube(g.n)));
        in.read(reinterpret_cast<char*>(g.values.data()), expected);
        if (!in) io_failure("failed while reading " + path);
    }
    check_grid(g);
    return g;
}

void save_grid(const Grid& g, const std::string& path) {
    check_grid(g);
    if (is_json_path(path)) {  // save_grid_json (voxel_io.cpp:84-95)
        std::string o = "{\"metadata\":" + metadata_json(g.metadata) + ",\"n\":" + std::to_string(g.n) + ",\"values\":[";
        o.reserve(o.size() + g.values.size() * 6);
        for (size_t k = 0; k < g.values.size(); ++k) {
            if (k) o += ',';
            json_double(o, g.values[k]);
        }
        o += "]}\n";
        write_file(path, o, "grid file");
        return;
    }
    // save_grid_raw (voxel_io.cpp:131-146): payload, then the sidecar
    write_file(path, std::string(reinterpret_cast<const char*>(g.values.data()), g.values.size() * sizeof(double)),
               "grid payload");
    write_file(path + ".json", "{\"metadata\":" + metadata_json(g.metadata) + ",\"n\":" + std::to_string(g.n) + "}\n",
               "grid sidecar");
}

Grid synthetic_sword(int n) {
    if (n < 8) throw FcctError(ST_INVALID_ARGUMENT, "synthetic_sword: n must be >= 8");
    const int c = std::max(1, n / 8);                                   // cross-section side
    const int hilt = std::max(1, static_cast<int>(std::lround(0.15 * n)));  // hilt length along x
    const int blade0 = hilt + 1;                                        // one-slab guard at x = hilt
    const int blade1 = std::min(n, blade0 + static_cast<int>(std::lround(0.7 * n)));
    const int y0 = (n - c) / 2, z0 = (n - c) / 2;
    const int gy0 = std::max(0, (n - 3 * c) / 2), gy1 = std::min(n, gy0 + 3 * c);
    Grid g;
    g.n = n;
    g.values.assign(static_cast<size_t>(cube(n)), 0.0);
    g.metadata["solid"] = "sword";
    auto fill = [&](int xa, int xb, int ya, int yb) {
        for (int x = xa; x < xb; ++x)
            for (int y = ya; y < yb; ++y)
                for (int z = z0; z < z0 + c; ++z) g.values[(static_cast<size_t>(x) * n + y) * n + z] = 1.0;
    };
    fill(0, hilt, y0, y0 + c);         // hilt
    fill(hilt, hilt + 1, gy0, gy1);    // cross-guard, three blades wide
    fill(blade0, blade1, y0, y0 + c);  // blade
    double filled = 0;
    for (const double v : g.values) filled += v;
    const double occ = filled / static_cast<double>(cube(n));
    if (!(occ > 0.0 && occ < 0.5)) throw std::logic_error("synthetic_sword occupancy out of range");
    return g;
}

uint64_t occupancy_checksum(const double* values, int64_t count) {
    uint64_t h = 14695981039346656037ULL;  // FNV-1a 64 offset basis
    for (int64_t i = 0; i < count; ++i) {
        h ^= static_cast<unsigned char>(values[i] != 0.0 ? '1' : '0');
        h *= 1099511628211ULL;
    }
    return h;
}

std::string spectrum_csv(int n, const Params& p, const std::complex<double>* values) {
    check_nodes(n, p);  // skew_nodes (spectral.cpp:155-171) runs the degeneracy check
    const auto xyz = node_coords(n, p);
    const int64_t N = cube(n);
    std::string head = "# n=" + std::to_string(n) + " params=" + encode_params(p) + "\n" + kSpectrumColumns + "\n";
    std::vector<std::string> parts(static_cast<size_t>(std::max(1, hw_threads())));
    std::vector<std::exception_ptr> errs(parts.size());
    parallel_chunks(N, 4096, [&](int64_t b, int64_t e, int t) {
        try {
            std::string& o = parts[static_cast<size_t>(t)];
            o.reserve(static_cast<size_t>((e - b) * 140));
            char buf[512];
            for (int64_t a = b; a < e; ++a) {
                const auto c = real_coords(xyz[static_cast<size_t>(a)]);
                const std::complex<double> v = values[a];
                const int i = static_cast<int>(a / (static_cast<int64_t>(n) * n)), j = static_cast<int>((a / n) % n),
                          k = static_cast<int>(a % n);
                const int len = std::snprintf(buf, sizeof(buf), "%d,%d,%d,%.17g,%.17g,%.17g,%.17g,%.17g,%.17g\n", i, j,
                                              k, c[0], c[1], c[2], v.real(), v.imag(), std::abs(v));
                o.append(buf, static_cast<size_t>(len));
            }
        } catch (...) {
            errs[static_cast<size_t>(t)] = std::current_exception();
        }
    });
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    size_t total = head.size();
    for (auto& s : parts) total += s.size();
    head.reserve(total);
    for (auto& s : parts) head += s;
    return head;
}

SpectrumFile load_spectrum_csv(const std::string& path, bool header_only) {
    std::ifstream probe(path, std::ios::binary);
    if (!probe) io_failure("cannot open spectrum file " + path);
    probe.close();
    const std::string text = read_file(path, "spectrum file");
    // split into getline()-style lines
    std::vector<std::pair<size_t, size_t>> lines;
    for (size_t pos = 0; pos < text.size();) {
        const size_t nl = text.find('\n', pos);
        const size_t e = nl == std::string::npos ? text.size() : nl;
        lines.emplace_back(pos, e - pos);
        pos = nl == std::string::npos ? text.size() : nl + 1;
    }
    auto line_at = [&](size_t k) { return text.substr(lines[k].first, lines[k].second); };
    SpectrumFile f;
    if (lines.empty() || line_at(0).rfind("# n=", 0) != 0)
        malformed("spectrum file lacks the '# n=... params=...' header");
    const std::string h = line_at(0);
    const auto pp = h.find(" params=");
    if (pp == std::string::npos) malformed("spectrum header lacks params");
    try {
        if (!stoi_like(h.substr(4, pp - 4), f.n)) throw std::invalid_argument("n");
        f.p = parse_params(h.substr(pp + 8));
    } catch (const std::exception&) {
        malformed("cannot parse spectrum header '" + h + "'");
    }
    if (f.n < 1 || f.n > 4096) malformed("spectrum header size out of range");
    if (lines.size() < 2 || line_at(1) != kSpectrumColumns) malformed("spectrum file lacks the column header");
    if (header_only) return f;

    const int64_t n3 = cube(f.n);
    // per-row parse in parallel; errors and duplicates resolved in row order
    enum : int8_t { RS_EMPTY, RS_OK, RS_FEW, RS_INT, RS_RANGE, RS_VAL };
    const int64_t nl = static_cast<int64_t>(lines.size()) - 2;
    std::vector<int8_t> st(static_cast<size_t>(std::max<int64_t>(nl, 0)));
    std::vector<int64_t> flat(st.size());
    std::vector<std::complex<double>> val(st.size());
    parallel_chunks(nl, 8192, [&](int64_t b, int64_t e, int) {
        std::string fields[9];
        for (int64_t r = b; r < e; ++r) {
            const auto [off, len] = lines[static_cast<size_t>(r + 2)];
            if (len == 0) {
                st[r] = RS_EMPTY;
                continue;
            }
            const std::string line = text.substr(off, len);
            size_t start = 0;
            bool few = false;
            for (int k = 0; k < 9; ++k) {
                const size_t end = k == 8 ? line.size() : line.find(',', start);
                if (end == std::string::npos) {
                    few = true;
                    break;
                }
                fields[k] = line.substr(start, end - start);
                start = end + 1;
            }
            if (few) {
                st[r] = RS_FEW;
                continue;
            }
            int i = 0, j = 0, k = 0;
            if (!stoi_like(fields[0], i) || !stoi_like(fields[1], j) || !stoi_like(fields[2], k)) {
                st[r] = RS_INT;
                continue;
            }
            if (i < 0 || i >= f.n || j < 0 || j >= f.n || k < 0 || k >= f.n) {
                st[r] = RS_RANGE;
                continue;
            }
            flat[r] = (static_cast<int64_t>(i) * f.n + j) * f.n + k;
            double re = 0, im = 0;
            st[r] = stod_like(fields[6], re) && stod_like(fields[7], im) ? RS_OK : RS_VAL;
            val[r] = {re, im};
        }
    });
    f.values.assign(static_cast<size_t>(n3), {0.0, 0.0});
    std::vector<uint8_t> seen(static_cast<size_t>(n3), 0);
    int64_t rows = 0;
    for (int64_t r = 0; r < nl; ++r) {
        const int8_t s = st[r];
        if (s == RS_EMPTY) continue;
        const std::string line = line_at(static_cast<size_t>(r + 2));
        if (s == RS_FEW) malformed("spectrum row has too few columns: " + line);
        if (s == RS_INT) malformed("cannot parse spectrum row: " + line);
        if (s == RS_RANGE) malformed("spectrum row index out of range: " + line);
        if (seen[flat[r]]) malformed("spectrum row repeats a node: " + line);
        seen[flat[r]] = 1;
        if (s == RS_VAL) malformed("cannot parse spectrum row: " + line);
        f.values[flat[r]] = val[r];
        ++rows;
    }
    if (rows != n3)
        throw FcctError(ST_SIZE_MISMATCH_IO, "spectrum file has " + std::to_string(rows) + " rows, header n=" +
                                                 std::to_string(f.n) + " requires " + std::to_string(n3));
    return f;
}

std::string nodes_csv(int n, const Params& p) {
    check_nodes(n, p);
    const auto xyz = node_coords(n, p);
    std::string o = "i,j,k,x,y,z\n";
    char buf[256];
    for (int64_t a = 0; a < cube(n); ++a) {
        const auto c = real_coords(xyz[static_cast<size_t>(a)]);
        const int len = std::snprintf(buf, sizeof(buf), "%d,%d,%d,%.17g,%.17g,%.17g\n",
                                      static_cast<int>(a / (static_cast<int64_t>(n) * n)), static_cast<int>((a / n) % n),
                                      static_cast<int>(a % n), c[0], c[1], c[2]);
        o.append(buf, static_cast<size_t>(len));
    }
    return o;
}

std::vector<Index3> shift_vectors() {
    std::set<Index3> out;
    for (const Index3 e : {Index3{1, 0, 0}, Index3{0, 1, 0}, Index3{0, 0, 1}})
        for (const auto& m : s4_group())
            out.insert(Index3{m[0] * e[0] + m[1] * e[1] + m[2] * e[2], m[3] * e[0] + m[4] * e[1] + m[5] * e[2],
                              m[6] * e[0] + m[7] * e[1] + m[8] * e[2]});
    return {out.begin(), out.end()};
}

std::string geometry_csv() {
    std::string o = "dx,dy,dz\n";
    for (const auto& v : shift_vectors())
        o += std::to_string(v[0]) + "," + std::to_string(v[1]) + "," + std::to_string(v[2]) + "\n";
    return o;
}

void write_text(const std::string& path, const std::string& content) {
    if (path.empty() || path == "-") {
        std::cout << content;
        std::cout.flush();
        return;
    }
    std::ofstream out(path, std::ios::trunc);
    if (!out) io_failure("cannot write " + path);
    out << content;
    if (!out) io_failure("failed while writing " + path);
}

}  // namespace fcct::io
