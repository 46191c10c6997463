// Mesh file ingestion: ASCII OFF and Wavefront OBJ, the formats and
// the error behaviour of the reference's load_mesh / write_mesh (src/mesh_io.cpp:32-115,
// 133-160), without a std::istringstream per line: the file is read in one block and
// parsed in place by one thread per chunk of lines, numbers with std::from_chars.
//
// Token rules follow the reference's stream extraction (libstdc++ num_get): a number is
// the longest run of characters its grammar accepts, and that whole run must convert
// ("1e" or "." is malformed, "1.5x" reads 1.5 and leaves "x" for the next field); a
// leading '+' is accepted for coordinates and counts, not for OBJ face indices (those
// go through from_chars in the reference too).  Conversions are correctly rounded in
// both (glibc strtod, from_chars), so coordinates are bit-identical.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <climits>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "mesh_host.hpp"

namespace gdb {
namespace {

[[noreturn]] void parse_fail(const std::string& path, const std::string& what) {
    throw std::runtime_error(path + ": " + what);
}

struct Cursor {
    const char* p;
    const char* e;  // end of the current line
};

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }

void skip_ws(Cursor& c) {
    while (c.p < c.e && is_ws(*c.p)) ++c.p;
}

// operator>>(double&) on the rest of the line
bool read_double(Cursor& c, double& out) {
    skip_ws(c);
    const char* s = c.p;
    const char* q = s;
    if (q < c.e && (*q == '+' || *q == '-')) ++q;
    const char* digits0 = q;
    while (q < c.e && std::isdigit(static_cast<unsigned char>(*q))) ++q;
    if (q < c.e && *q == '.') {
        ++q;
        while (q < c.e && std::isdigit(static_cast<unsigned char>(*q))) ++q;
    }
    const bool mant = q > digits0 && !(q - digits0 == 1 && *digits0 == '.');
    if (q < c.e && (*q == 'e' || *q == 'E') && mant) {
        ++q;
        if (q < c.e && (*q == '+' || *q == '-')) ++q;
        while (q < c.e && std::isdigit(static_cast<unsigned char>(*q))) ++q;
    }
    if (q == s) return false;
    const char* b = s;
    if (*b == '+') ++b;
    if (b < q && *b == '+') return false;
    double v = 0.0;
    const auto r = std::from_chars(b, q, v);
    if (r.ec != std::errc() || r.ptr != q) return false;  // the whole run must convert
    out = v;
    c.p = q;
    return true;
}

// operator>>(long long&) on the rest of the line
bool read_ll(Cursor& c, long long& out) {
    skip_ws(c);
    const char* s = c.p;
    const char* q = s;
    if (q < c.e && (*q == '+' || *q == '-')) ++q;
    const char* d0 = q;
    while (q < c.e && std::isdigit(static_cast<unsigned char>(*q))) ++q;
    if (q == d0) return false;
    const char* b = *s == '+' ? s + 1 : s;
    long long v = 0;
    const auto r = std::from_chars(b, q, v);
    if (r.ec != std::errc() || r.ptr != q) return false;
    out = v;
    c.p = q;
    return true;
}

bool read_token(Cursor& c, const char*& t0, const char*& t1) {
    skip_ws(c);
    if (c.p >= c.e) return false;
    t0 = c.p;
    while (c.p < c.e && !is_ws(*c.p)) ++c.p;
    t1 = c.p;
    return true;
}

struct Lines {
    const char* p;
    const char* end;
    // next line (without its '\n'); false at end of input
    bool next(Cursor& c) {
        if (p >= end) return false;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
        c.p = p;
        c.e = nl ? nl : end;
        p = nl ? nl + 1 : end;
        return true;
    }
    // next line that is not blank and does not start (after blanks) with '#'
    bool next_content(Cursor& c) {
        while (next(c)) {
            const char* q = c.p;
            while (q < c.e && (*q == ' ' || *q == '\t' || *q == '\r' || *q == '\n')) ++q;
            if (q == c.e || *q == '#') continue;
            return true;
        }
        return false;
    }
};

// The body of a file is cut into chunks at line boundaries and parsed by one thread
// per chunk in two passes: count the records of every chunk (content lines for OFF,
// v / f records for OBJ), then parse each chunk straight into the output arrays at its
// prefix offsets.  A chunk stops at its first bad record; the first chunk (in file
// order) that stopped names the error, so the message is the one the reference's
// sequential reader gives.
std::vector<Cursor> split_chunks(const char* b, const char* e) {
    const size_t len = static_cast<size_t>(e - b);
    unsigned hw = std::thread::hardware_concurrency();
    const unsigned T = len < (4u << 20) ? 1u : std::max(1u, std::min(hw ? hw : 1u, 32u));
    std::vector<Cursor> ch;
    const char* x = b;
    for (unsigned t = 0; t < T; ++t) {
        const char* y = t + 1 == T ? e : b + len * (t + 1) / T;
        if (y < x) y = x;
        if (y < e) {
            const char* nl = static_cast<const char*>(std::memchr(y, '\n', e - y));
            y = nl ? nl + 1 : e;
        }
        ch.push_back({x, y});
        x = y;
    }
    return ch;
}

template <typename Fn>
void parallel_for(size_t n, Fn&& fn) {
    if (n <= 1) {
        for (size_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(n);
    for (size_t i = 0; i < n; ++i) th.emplace_back([&fn, i] { fn(i); });
    for (auto& t : th) t.join();
}

void load_off(const std::string& path, const std::string& text, MeshData& m) {
    Lines L{text.data(), text.data() + text.size()};
    Cursor c;
    if (!L.next_content(c)) parse_fail(path, "empty OFF file");
    const char *t0, *t1;
    if (!read_token(c, t0, t1) || std::string(t0, t1) != "OFF") parse_fail(path, "missing OFF header");
    long long nv = -1, nf = -1, ne = 0;
    {
        long long a = -1, b = -1, e = 0;
        const bool ok = read_ll(c, a) && read_ll(c, b) && read_ll(c, e);
        if (ok) {
            nv = a; nf = b; ne = e;
        } else {
            if (!L.next_content(c)) parse_fail(path, "missing element counts");
            if (!(read_ll(c, nv) && read_ll(c, nf) && read_ll(c, ne)))
                parse_fail(path, "malformed element counts");
        }
    }
    (void)ne;
    if (nv < 0 || nf < 0) parse_fail(path, "negative element counts");
    const std::vector<Cursor> ch = split_chunks(L.p, L.end);
    const size_t C = ch.size();
    // pass 1: content lines per chunk
    std::vector<long long> cnt(C + 1, 0);
    parallel_for(C, [&](size_t k) {
        Lines l{ch[k].p, ch[k].e};
        Cursor x;
        long long n = 0;
        while (l.next_content(x)) ++n;
        cnt[k + 1] = n;
    });
    for (size_t k = 0; k < C; ++k) cnt[k + 1] += cnt[k];
    const long long total = cnt[C];
    const long long nv_have = std::min(total, nv);
    const long long nf_have = std::max(0LL, std::min(total - nv, nf));
    m.xyz.assign(3 * static_cast<size_t>(nv_have), 0.0);
    m.faces.assign(3 * static_cast<size_t>(nf_have), 0);
    // pass 2: parse; err_at = global content-line index of the chunk's first bad line
    std::vector<long long> err_at(C, -1), err_k(C, 0);
    parallel_for(C, [&](size_t k) {
        Lines l{ch[k].p, ch[k].e};
        Cursor x;
        for (long long g = cnt[k]; g < nv + nf && l.next_content(x); ++g) {
            if (g < nv) {
                double a, b, d;
                if (!(read_double(x, a) && read_double(x, b) && read_double(x, d))) {
                    err_at[k] = g;
                    return;
                }
                double* o = &m.xyz[3 * static_cast<size_t>(g)];
                o[0] = a; o[1] = b; o[2] = d;
            } else {
                long long kk, a, b, d;
                if (!read_ll(x, kk)) {
                    err_at[k] = g;
                    err_k[k] = LLONG_MIN;
                    return;
                }
                if (kk != 3 || !(read_ll(x, a) && read_ll(x, b) && read_ll(x, d))) {
                    err_at[k] = g;
                    err_k[k] = kk;
                    return;
                }
                int32_t* o = &m.faces[3 * static_cast<size_t>(g - nv)];
                o[0] = static_cast<int32_t>(a);
                o[1] = static_cast<int32_t>(b);
                o[2] = static_cast<int32_t>(d);
            }
        }
    });
    for (size_t k = 0; k < C; ++k) {
        const long long g = err_at[k];
        if (g < 0) continue;
        if (g < nv) parse_fail(path, "malformed vertex " + std::to_string(g));
        const long long f = g - nv;
        if (err_k[k] == LLONG_MIN || err_k[k] == 3) parse_fail(path, "malformed face " + std::to_string(f));
        parse_fail(path, "face " + std::to_string(f) + " has " + std::to_string(err_k[k]) +
                             " vertices, only triangles are supported");
    }
    if (total < nv) parse_fail(path, "unexpected end of file in vertex " + std::to_string(total));
    if (total < nv + nf)
        parse_fail(path, "unexpected end of file in face " + std::to_string(total - nv));
}

int32_t obj_corner_index(const char* t0, const char* t1, size_t nv, const std::string& path,
                         long long record) {
    const char* slash = static_cast<const char*>(std::memchr(t0, '/', t1 - t0));
    const char* h1 = slash ? slash : t1;
    long long idx = 0;
    const auto r = std::from_chars(t0, h1, idx);
    if (r.ec != std::errc() || r.ptr != h1)
        parse_fail(path, "malformed face index '" + std::string(t0, t1) + "' in f record " +
                             std::to_string(record));
    if (idx < 0) idx += static_cast<long long>(nv) + 1;  // OBJ relative indexing
    if (idx < 1) parse_fail(path, "face index out of range in f record " + std::to_string(record));
    return static_cast<int32_t>(idx - 1);
}

// 'v' / 'f' / other for the line's first token
inline int obj_tag(Cursor& x) {
    const char *t0, *t1;
    if (!read_token(x, t0, t1) || t1 - t0 != 1) return 0;
    return *t0 == 'v' ? 1 : *t0 == 'f' ? 2 : 0;
}

void load_obj(const std::string& path, const std::string& text, MeshData& m) {
    const std::vector<Cursor> ch = split_chunks(text.data(), text.data() + text.size());
    const size_t C = ch.size();
    std::vector<long long> nvk(C + 1, 0), nfk(C + 1, 0);
    parallel_for(C, [&](size_t k) {
        Lines l{ch[k].p, ch[k].e};
        Cursor x;
        long long a = 0, b = 0;
        while (l.next(x)) {
            const int t = obj_tag(x);
            a += t == 1;
            b += t == 2;
        }
        nvk[k + 1] = a;
        nfk[k + 1] = b;
    });
    for (size_t k = 0; k < C; ++k) {
        nvk[k + 1] += nvk[k];
        nfk[k + 1] += nfk[k];
    }
    m.xyz.assign(3 * static_cast<size_t>(nvk[C]), 0.0);
    m.faces.assign(3 * static_cast<size_t>(nfk[C]), 0);
    std::vector<std::string> err(C);
    parallel_for(C, [&](size_t k) {
        Lines l{ch[k].p, ch[k].e};
        Cursor x;
        long long v = nvk[k], f = nfk[k];
        try {
            while (l.next(x)) {
                const int t = obj_tag(x);
                if (t == 1) {
                    double a, b, d;
                    if (!(read_double(x, a) && read_double(x, b) && read_double(x, d)))
                        parse_fail(path, "malformed v record " + std::to_string(v));
                    double* o = &m.xyz[3 * static_cast<size_t>(v)];
                    o[0] = a; o[1] = b; o[2] = d;
                    ++v;
                } else if (t == 2) {
                    const char* tok[3][2];
                    int cnt = 0;
                    const char *a0, *a1;
                    while (read_token(x, a0, a1)) {
                        if (cnt < 3) {
                            tok[cnt][0] = a0;
                            tok[cnt][1] = a1;
                        }
                        ++cnt;
                    }
                    if (cnt != 3)
                        parse_fail(path, "f record " + std::to_string(f) + " has " +
                                             std::to_string(cnt) +
                                             " corners, only triangles are supported");
                    int32_t* o = &m.faces[3 * static_cast<size_t>(f)];
                    for (int q = 0; q < 3; ++q)
                        o[q] = obj_corner_index(tok[q][0], tok[q][1], static_cast<size_t>(v), path, f);
                    ++f;
                }
                // vt / vn / usemtl / ... records are ignored
            }
        } catch (const std::runtime_error& e) {
            err[k] = e.what();
        }
    });
    for (size_t k = 0; k < C; ++k)
        if (!err[k].empty()) throw std::runtime_error(err[k]);
}

}  // namespace

void load_mesh_file(const std::string& path, MeshData& m) {
    const auto dot = path.find_last_of('.');
    std::string ext = dot == std::string::npos ? "" : path.substr(dot + 1);
    std::transform(ext.begin(), ext.end(), ext.begin(),
                   [](unsigned char ch) { return static_cast<char>(std::tolower(ch)); });
    if (ext != "off" && ext != "obj")
        throw std::runtime_error(path + ": unsupported mesh format '." + ext + "' (use .off or .obj)");
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error(path + ": cannot open file");
    std::string text;
    std::fseek(f, 0, SEEK_END);
    const long size = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    if (size > 0) {
        text.resize(static_cast<size_t>(size));
        const size_t got = std::fread(&text[0], 1, text.size(), f);
        text.resize(got);
    }
    std::fclose(f);
    if (ext == "off")
        load_off(path, text, m);
    else
        load_obj(path, text, m);
    if (m.xyz.size() / 3 > static_cast<size_t>(INT32_MAX) || m.faces.size() / 3 > static_cast<size_t>(INT32_MAX))
        throw std::runtime_error(path + ": mesh too large for int32 indices");
    try {
        validate(m.xyz.data(), static_cast<int32_t>(m.xyz.size() / 3), m.faces.data(),
                 static_cast<int32_t>(m.faces.size() / 3));
    } catch (const std::runtime_error& e) {
        throw std::runtime_error(path + ": " + e.what());
    }
}

void write_mesh_file(const std::string& path, const double* xyz, int32_t n, const int32_t* faces,
                     int32_t nf, bool off) {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error(path + ": cannot open file for writing");
    std::string buf;
    buf.reserve(1 << 20);
    char num[64];
    auto flush = [&] {
        if (!buf.empty() && std::fwrite(buf.data(), 1, buf.size(), f) != buf.size()) {
            std::fclose(f);
            throw std::runtime_error(path + ": write failed");
        }
        buf.clear();
    };
    auto coord = [&](double v) {  // "%.17g": loading the file back is bit-exact
        const int k = std::snprintf(num, sizeof num, "%.17g", v);
        buf.append(num, static_cast<size_t>(k));
    };
    if (off) {
        buf += "OFF\n" + std::to_string(n) + ' ' + std::to_string(nf) + " 0\n";
        for (int32_t v = 0; v < n; ++v) {
            coord(xyz[3 * static_cast<size_t>(v)]);
            buf += ' ';
            coord(xyz[3 * static_cast<size_t>(v) + 1]);
            buf += ' ';
            coord(xyz[3 * static_cast<size_t>(v) + 2]);
            buf += '\n';
            if (buf.size() > (1 << 20)) flush();
        }
        for (int32_t t = 0; t < nf; ++t) {
            const int32_t* x = faces + 3 * static_cast<size_t>(t);
            buf += "3 " + std::to_string(x[0]) + ' ' + std::to_string(x[1]) + ' ' + std::to_string(x[2]) + '\n';
            if (buf.size() > (1 << 20)) flush();
        }
    } else {
        for (int32_t v = 0; v < n; ++v) {
            buf += "v ";
            coord(xyz[3 * static_cast<size_t>(v)]);
            buf += ' ';
            coord(xyz[3 * static_cast<size_t>(v) + 1]);
            buf += ' ';
            coord(xyz[3 * static_cast<size_t>(v) + 2]);
            buf += '\n';
            if (buf.size() > (1 << 20)) flush();
        }
        for (int32_t t = 0; t < nf; ++t) {
            const int32_t* x = faces + 3 * static_cast<size_t>(t);
            buf += "f " + std::to_string(x[0] + 1) + ' ' + std::to_string(x[1] + 1) + ' ' +
                   std::to_string(x[2] + 1) + '\n';
            if (buf.size() > (1 << 20)) flush();
        }
    }
    flush();
    if (std::fclose(f) != 0) throw std::runtime_error(path + ": write failed");
}

}  // namespace gdb
