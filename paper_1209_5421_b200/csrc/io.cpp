// io.cpp — the reference's file readers, host side:
//   aux_read_matrix_market  <- read_matrix_market  matrix_market.hpp:33-104
//   aux_read_mesh           <- read_mesh           problems.hpp:201-310
//   aux_read_coords         <- read_coords         problems.hpp:313-330
//   aux_write_matrix_market <- write_matrix_market matrix_market.hpp:106-120
//
// The file is read into memory once and its lines are parsed by several host
// threads (each takes a contiguous byte range starting at a line boundary and
// keeps its entries in order); a prefix over the per-range line counts gives
// the 1-based line numbers, so the FIRST error in file order is reported with
// the reference's message and line number (parse_error, errors.hpp:67-76).
// Entries keep the file order, and csr_from_triplets (sparse.hpp:193-215) is a
// stable counting sort by row then a stable sort by column inside each row,
// duplicates summed from 0.0 in file order — the reference sorts with the
// unstable std::sort, so only a file that repeats an entry can differ (in the
// last bit of that entry's sum).  Numbers are parsed like the reference's
// istream extraction: integers as `long` (sign, digits), reals by the
// num_get grammar handed to strtod (correctly rounded, overflow rejected).
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/auxamg_b200.h"

namespace {

struct AuxIoError : std::runtime_error {
    aux_status st;
    AuxIoError(aux_status s, const std::string& w) : std::runtime_error(w), st(s) {}
};
[[noreturn]] void io_fail(const std::string& w) { throw AuxIoError(AUX_IO_ERROR, w); }
[[noreturn]] void parse_fail(const std::string& w, long line) {
    throw AuxIoError(AUX_PARSE_ERROR, w + " (line " + std::to_string(line) + ")");
}

std::vector<char> slurp(const char* path) {
    FILE* f = std::fopen(path, "rb");
    if (!f) io_fail(std::string("cannot open ") + path);
    std::vector<char> buf;
    std::fseek(f, 0, SEEK_END);
    const long sz = std::ftell(f);
    if (sz < 0) {
        std::fclose(f);
        io_fail(std::string("cannot open ") + path);
    }
    std::fseek(f, 0, SEEK_SET);
    buf.resize((size_t)sz + 1);
    const size_t got = std::fread(buf.data(), 1, (size_t)sz, f);
    std::fclose(f);
    if (got != (size_t)sz) io_fail(std::string("cannot open ") + path);
    buf[(size_t)sz] = '\0';
    buf.resize((size_t)sz);   // data()[size()] stays '\0' (capacity kept)
    return buf;
}

int pick_threads(int t) {
    if (t > 0) return t;
    const unsigned h = std::thread::hardware_concurrency();
    return h ? (int)std::min(h, 64u) : 1;
}

// Line cursor with std::getline semantics: a final line without '\n' counts,
// a trailing '\n' adds no empty line.
struct Cursor {
    const char* p;
    const char* end;
    bool next(const char*& b, const char*& e) {
        if (p >= end) return false;
        b = p;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(end - p)));
        e = nl ? nl : end;
        p = nl ? nl + 1 : end;
        return true;
    }
};

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }
inline bool blank(const char* b, const char* e) {   // find_first_not_of(" \t\r") == npos
    for (; b < e; ++b)
        if (*b != ' ' && *b != '\t' && *b != '\r') return false;
    return true;
}

// `is >> long`: skip white space, optional sign, at least one digit
bool get_long(const char*& p, const char* e, long& out) {
    while (p < e && is_ws(*p)) ++p;
    const char* q = p;
    bool neg = false;
    if (q < e && (*q == '+' || *q == '-')) neg = *q++ == '-';
    if (q >= e || !std::isdigit((unsigned char)*q)) return false;
    unsigned long long v = 0;
    while (q < e && std::isdigit((unsigned char)*q)) {
        v = v * 10 + (unsigned)(*q++ - '0');
        if (v > (unsigned long long)9223372036854775807ll + (neg ? 1 : 0)) return false;
    }
    out = neg ? (long)(0 - v) : (long)v;
    p = q;
    return true;
}

// `is >> double`: the num_get grammar [sign] digits [. digits] [e [sign] digits]
// collected, then strtod; overflow to +-inf fails like libstdc++'s conversion
bool get_double(const char*& p, const char* e, double& out) {
    while (p < e && is_ws(*p)) ++p;
    const char* q = p;
    char tok[400];
    int n = 0;
    auto put = [&](char c) { if (n < (int)sizeof tok - 1) tok[n++] = c; };
    if (q < e && (*q == '+' || *q == '-')) put(*q++);
    bool digits = false;
    while (q < e && std::isdigit((unsigned char)*q)) { put(*q++); digits = true; }
    if (q < e && *q == '.') {
        put(*q++);
        while (q < e && std::isdigit((unsigned char)*q)) { put(*q++); digits = true; }
    }
    if (!digits) return false;
    if (q < e && (*q == 'e' || *q == 'E')) {
        put(*q++);
        if (q < e && (*q == '+' || *q == '-')) put(*q++);
        bool ed = false;
        while (q < e && std::isdigit((unsigned char)*q)) { put(*q++); ed = true; }
        if (!ed) return false;   // "1e" does not convert completely
    }
    tok[n] = '\0';
    char* s = nullptr;
    const double v = std::strtod(tok, &s);
    if (s != tok + n || std::isinf(v)) return false;
    out = v;
    p = q;
    return true;
}

// Parallel pass over the lines of [b, e): every range starts at a line start;
// fn(range, line_begin, line_end, local_line) is called for each line in order.
template <class Fn>
void parallel_lines(const char* b, const char* e, int threads, std::vector<long>& lines_per_range, Fn fn) {
    const size_t len = (size_t)(e - b);
    int T = std::max(1, std::min(threads, (int)(len / (1 << 16)) + 1));
    std::vector<const char*> cut(T + 1);
    cut[0] = b;
    cut[T] = e;
    for (int t = 1; t < T; ++t) {
        const char* c = b + len * t / T;
        if (c < cut[t - 1]) c = cut[t - 1];
        const char* nl = static_cast<const char*>(std::memchr(c, '\n', (size_t)(e - c)));
        cut[t] = nl ? nl + 1 : e;
    }
    lines_per_range.assign(T, 0);
    auto work = [&](int t) {
        Cursor cur{cut[t], cut[t + 1]};
        const char *lb, *le;
        long k = 0;
        while (cur.next(lb, le)) fn(t, lb, le, k++);
        lines_per_range[t] = k;
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
}

std::string lower(std::string s) {
    for (char& c : s) c = (char)std::tolower((unsigned char)c);
    return s;
}

std::vector<std::string> words(const char* b, const char* e, int max_words) {
    std::vector<std::string> w;
    const char* p = b;
    while ((int)w.size() < max_words) {
        while (p < e && is_ws(*p)) ++p;
        if (p >= e) break;
        const char* q = p;
        while (q < e && !is_ws(*q)) ++q;
        w.emplace_back(p, q);
        p = q;
    }
    return w;
}

}  // namespace

struct aux_file_data {
    int kind = 0;   // 0 CSR, 1 mesh, 2 coords
    int64_t a = 0, b = 0, c = 0;
    std::vector<int32_t> i0, i1;
    std::vector<double> d0;
};

namespace {

// csr_from_triplets (sparse.hpp:193-215) over in-order triplets
void build_csr(aux_file_data* D, long n_rows, long n_cols, const std::vector<int32_t>& r, const std::vector<int32_t>& c,
               const std::vector<double>& v, int threads) {
    const size_t m = r.size();
    std::vector<int64_t> start((size_t)n_rows + 1, 0);
    for (size_t k = 0; k < m; ++k) ++start[(size_t)r[k] + 1];
    for (long i = 0; i < n_rows; ++i) start[(size_t)i + 1] += start[(size_t)i];
    std::vector<int64_t> pos(start.begin(), start.end() - 1);
    std::vector<int32_t> sc(m);
    std::vector<double> sv(m);
    for (size_t k = 0; k < m; ++k) {   // stable by row: file order within a row
        const int64_t q = pos[(size_t)r[k]]++;
        sc[(size_t)q] = c[k];
        sv[(size_t)q] = v[k];
    }
    // per row: stable sort by column, duplicates summed from 0.0 in order
    std::vector<int32_t> cnt((size_t)n_rows, 0);
    const int T = std::max(1, std::min(threads, (int)(n_rows / 4096) + 1));
    auto sort_rows = [&](int t) {
        std::vector<int> ord;
        std::vector<int32_t> tc;
        std::vector<double> tv;
        for (long i = n_rows * t / T; i < n_rows * (t + 1) / T; ++i) {
            const int64_t s0 = start[(size_t)i], s1 = start[(size_t)i + 1];
            const int len = (int)(s1 - s0);
            ord.resize(len);
            std::iota(ord.begin(), ord.end(), 0);
            std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return sc[s0 + x] < sc[s0 + y]; });
            tc.assign(sc.begin() + s0, sc.begin() + s1);
            tv.assign(sv.begin() + s0, sv.begin() + s1);
            int w = 0;
            for (int k = 0; k < len;) {
                int j = k;
                double sum = 0.0;
                while (j < len && tc[ord[j]] == tc[ord[k]]) sum += tv[ord[j++]];
                sc[s0 + w] = tc[ord[k]];
                sv[s0 + w] = sum;
                ++w;
                k = j;
            }
            cnt[(size_t)i] = w;
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(sort_rows, t);
    sort_rows(0);
    for (auto& x : th) x.join();
    D->kind = 0;
    D->a = n_rows;
    D->b = n_cols;
    D->i0.assign((size_t)n_rows + 1, 0);
    for (long i = 0; i < n_rows; ++i) D->i0[(size_t)i + 1] = D->i0[(size_t)i] + cnt[(size_t)i];
    const int64_t nnz = D->i0[(size_t)n_rows];
    D->c = nnz;
    D->i1.resize((size_t)nnz);
    D->d0.resize((size_t)nnz);
    for (long i = 0; i < n_rows; ++i) {
        std::copy(sc.begin() + start[(size_t)i], sc.begin() + start[(size_t)i] + cnt[(size_t)i], D->i1.begin() + D->i0[(size_t)i]);
        std::copy(sv.begin() + start[(size_t)i], sv.begin() + start[(size_t)i] + cnt[(size_t)i], D->d0.begin() + D->i0[(size_t)i]);
    }
}

struct LineErr {
    long line = -1;   // range-local line index, -1: none
    std::string what;
};

void read_mm(const char* path, int threads, aux_file_data* D) {
    const std::vector<char> buf = slurp(path);
    Cursor cur{buf.data(), buf.data() + buf.size()};
    const char *lb, *le;
    long line_no = 0;
    if (!cur.next(lb, le)) parse_fail("empty file", 1);
    ++line_no;
    const auto h = words(lb, le, 5);
    auto w = [&](size_t i) { return i < h.size() ? h[i] : std::string(); };
    if (w(0) != "%%MatrixMarket" || lower(w(1)) != "matrix") parse_fail("not a Matrix Market matrix file", line_no);
    if (lower(w(2)) != "coordinate") parse_fail("only coordinate format is supported", line_no);
    if (lower(w(3)) != "real") parse_fail("only real-valued matrices are supported", line_no);
    const std::string sym = lower(w(4));
    if (sym != "general" && sym != "symmetric") parse_fail("symmetry must be general or symmetric", line_no);
    long n_rows = 0, n_cols = 0, nnz = 0;
    for (;;) {
        if (!cur.next(lb, le)) parse_fail("missing size line", line_no);
        ++line_no;
        if (lb == le || lb[0] == '%') continue;
        const char* p = lb;
        if (!get_long(p, le, n_rows) || !get_long(p, le, n_cols) || !get_long(p, le, nnz) || n_rows < 0 || n_cols < 0 ||
            nnz < 0)
            parse_fail("malformed size line", line_no);
        break;
    }
    const bool symm = sym == "symmetric";
    // entries: per range, in file order
    const int T0 = pick_threads(threads);
    std::vector<std::vector<int32_t>> er(T0 + 1), ec(T0 + 1);
    std::vector<std::vector<double>> ev(T0 + 1);
    std::vector<std::vector<long>> eline(T0 + 1);   // range-local line of each entry
    std::vector<LineErr> err(T0 + 1);
    std::vector<long> lines;
    parallel_lines(cur.p, cur.end, T0, lines, [&](int t, const char* b, const char* e, long k) {
        if (err[t].line >= 0) return;
        if (b == e || b[0] == '%') return;
        const char* p = b;
        long r = 0, c = 0;
        double v = 0.0;
        if (!get_long(p, e, r) || !get_long(p, e, c) || !get_double(p, e, v)) {
            err[t] = {k, "malformed entry"};
            return;
        }
        if (r < 1 || r > n_rows || c < 1 || c > n_cols) {
            err[t] = {k, "index out of range (indices are 1-based)"};
            return;
        }
        er[t].push_back((int32_t)(r - 1));
        ec[t].push_back((int32_t)(c - 1));
        ev[t].push_back(v);
        eline[t].push_back(k);
    });
    // the reference stops after nnz entries: an error counts only before that
    const int T = (int)lines.size();
    long seen = 0, base = line_no;
    std::vector<int32_t> R, C;
    std::vector<double> V;
    R.reserve((size_t)(symm ? 2 * nnz : nnz));
    C.reserve(R.capacity());
    V.reserve(R.capacity());
    for (int t = 0; t < T && seen < nnz; ++t) {
        const long take = std::min<long>((long)er[t].size(), nnz - seen);
        for (long k = 0; k < take; ++k) {
            R.push_back(er[t][k]);
            C.push_back(ec[t][k]);
            V.push_back(ev[t][k]);
            if (symm && er[t][k] != ec[t][k]) {
                R.push_back(ec[t][k]);
                C.push_back(er[t][k]);
                V.push_back(ev[t][k]);
            }
        }
        seen += take;
        if (seen < nnz && err[t].line >= 0) parse_fail(err[t].what, base + err[t].line + 1);
        base += lines[t];
    }
    if (seen < nnz)
        parse_fail("file ends after " + std::to_string(seen) + " of " + std::to_string(nnz) + " entries", base);
    if (n_rows > 2147483647l || n_cols > 2147483647l) throw AuxIoError(AUX_SIZE_ERROR, "matrix too large for int32 CSR");
    build_csr(D, n_rows, n_cols, R, C, V, T0);
}

// Next non-blank line (problems.hpp:207-213 next_line)
struct LineReader {
    Cursor cur;
    long line_no = 0;
    const char *b = nullptr, *e = nullptr;
    void next(const char* what) {
        for (;;) {
            if (!cur.next(b, e)) parse_fail(std::string("missing ") + what, line_no);
            ++line_no;
            if (!blank(b, e)) return;
        }
    }
};

// the next `count` non-blank lines, parsed in parallel by fn(index, b, e, msg)
// (false + message on a malformed line).  Returns the index of the first bad
// line in file order (or count) with its message; ln receives every line's
// 1-based number.
template <class Fn>
long parse_block(LineReader& L, long count, const char* what, int threads, std::vector<long>& ln, std::string& msg,
                 Fn fn) {
    std::vector<const char*> lb((size_t)count), le((size_t)count);
    ln.assign((size_t)count, 0);
    for (long i = 0; i < count; ++i) {
        L.next(what);
        lb[(size_t)i] = L.b;
        le[(size_t)i] = L.e;
        ln[(size_t)i] = L.line_no;
    }
    const int T = std::max(1, std::min(pick_threads(threads), (int)(count / 8192) + 1));
    std::vector<long> bad(T, -1);
    std::vector<std::string> m(T);
    auto work = [&](int t) {
        for (long i = count * t / T; i < count * (t + 1) / T; ++i)
            if (!fn(i, lb[(size_t)i], le[(size_t)i], m[t])) {
                bad[t] = i;
                return;
            }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    for (int t = 0; t < T; ++t)
        if (bad[t] >= 0) {
            msg = m[t];
            return bad[t];
        }
    return count;
}

// ids[0 .. upto): the first repeated id in file order (its index), or upto
long first_duplicate(const std::vector<long>& ids, long upto, long range) {
    std::vector<char> seen((size_t)range, 0);
    for (long i = 0; i < upto; ++i) {
        if (seen[(size_t)ids[(size_t)i] - 1]) return i;
        seen[(size_t)ids[(size_t)i] - 1] = 1;
    }
    return upto;
}

void read_mesh_file(const char* path, int threads, aux_file_data* D) {
    const std::vector<char> buf = slurp(path);
    LineReader L{Cursor{buf.data(), buf.data() + buf.size()}};
    L.next("NODES header");
    long count = 0;
    {
        const auto w = words(L.b, L.e, 1);
        const char* p = L.b;
        while (p < L.e && is_ws(*p)) ++p;
        while (p < L.e && !is_ws(*p)) ++p;
        if (w.empty() || w[0] != "NODES" || !get_long(p, L.e, count) || count < 1)
            parse_fail("expected 'NODES <count>'", L.line_no);
    }
    const long nn = count;
    std::vector<double> xy(2 * (size_t)nn, 0.0);
    // lines parsed in parallel; the first problem in file order (a malformed
    // line or a repeated id) is reported, as the sequential reference does
    std::vector<long> ids((size_t)nn), ln;
    std::string msg;
    const long bad = parse_block(L, nn, "node line", threads, ln, msg, [&](long i, const char* b, const char* e, std::string& m) {
        const char* p = b;
        long id = 0;
        double x = 0.0, y = 0.0;
        if (!get_long(p, e, id) || !get_double(p, e, x) || !get_double(p, e, y)) { m = "malformed node line"; return false; }
        if (id < 1 || id > nn) { m = "node id out of range (ids are 1-based)"; return false; }
        ids[(size_t)i] = id;
        xy[2 * (size_t)(id - 1)] = x;
        xy[2 * (size_t)(id - 1) + 1] = y;
        return true;
    });
    {
        const long dup = first_duplicate(ids, bad, nn);
        if (dup < bad) parse_fail("duplicate node id", ln[(size_t)dup]);
        if (bad < nn) parse_fail(msg, ln[(size_t)bad]);
    }
    L.next("ELEMENTS header");
    {
        const auto w = words(L.b, L.e, 1);
        const char* p = L.b;
        while (p < L.e && is_ws(*p)) ++p;
        while (p < L.e && !is_ws(*p)) ++p;
        if (w.empty() || w[0] != "ELEMENTS" || !get_long(p, L.e, count) || count < 1)
            parse_fail("expected 'ELEMENTS <count>'", L.line_no);
    }
    const long ne = count;
    std::vector<int32_t> tri(3 * (size_t)ne, 0);
    std::vector<long> eids((size_t)ne);
    const long ebad = parse_block(L, ne, "element line", threads, ln, msg, [&](long i, const char* b, const char* e, std::string& m) {
        const char* p = b;
        long id = 0, v[3] = {0, 0, 0};
        if (!get_long(p, e, id) || !get_long(p, e, v[0]) || !get_long(p, e, v[1]) || !get_long(p, e, v[2])) {
            m = "malformed element line";
            return false;
        }
        if (id < 1 || id > ne) { m = "element id out of range (ids are 1-based)"; return false; }
        eids[(size_t)i] = id;   // (a repeated id is checked in file order below, before the vertices)
        for (int s = 0; s < 3; ++s)
            if (v[s] < 1 || v[s] > nn) { m = "vertex index out of range (ids are 1-based)"; return false; }
        for (int s = 0; s < 3; ++s) tri[3 * (size_t)(id - 1) + s] = (int32_t)(v[s] - 1);
        return true;
    });
    {
        // a repeated id is rejected before its vertices are checked (problems.hpp:250-255):
        // line `ebad` itself counts when its id was parsed and repeats an earlier one
        long upto = ebad;
        if (ebad < ne && msg == "vertex index out of range (ids are 1-based)") upto = ebad + 1;
        const long dup = first_duplicate(eids, upto, ne);
        if (dup < upto) parse_fail("duplicate element id", ln[(size_t)dup]);
        if (ebad < ne) parse_fail(msg, ln[(size_t)ebad]);
    }
    // optional BOUNDARY section
    std::vector<int32_t> bnd;
    {
        const char *b = nullptr, *e = nullptr;
        bool more = false;
        while (L.cur.next(b, e)) {
            ++L.line_no;
            if (!blank(b, e)) {
                more = true;
                break;
            }
        }
        if (more) {
            const char* p = b;
            while (p < e && is_ws(*p)) ++p;
            const char* q = p;
            while (q < e && !is_ws(*q)) ++q;
            if (std::string(p, q) != "BOUNDARY") parse_fail("expected 'BOUNDARY <count>'", L.line_no);
            long bc = 0;
            if (!get_long(q, e, bc) || bc < 0) parse_fail("expected 'BOUNDARY <count>'", L.line_no);
            long got = 0;
            while (got < bc) {
                L.next("boundary ids");
                const char* r = L.b;
                long id = 0;
                while (got < bc && get_long(r, L.e, id)) {
                    if (id < 1 || id > nn) parse_fail("boundary node id out of range", L.line_no);
                    bnd.push_back((int32_t)(id - 1));
                    ++got;
                }
            }
        }
    }
    // free boundary: endpoints of edges used by exactly one triangle
    {
        std::vector<uint64_t> edges(3 * (size_t)ne);
        for (long t = 0; t < ne; ++t)
            for (int s = 0; s < 3; ++s) {
                const uint32_t a = (uint32_t)tri[3 * (size_t)t + s], b = (uint32_t)tri[3 * (size_t)t + (s + 1) % 3];
                edges[3 * (size_t)t + s] = ((uint64_t)std::min(a, b) << 32) | std::max(a, b);
            }
        std::sort(edges.begin(), edges.end());
        for (size_t i = 0; i < edges.size();) {
            size_t j = i;
            while (j < edges.size() && edges[j] == edges[i]) ++j;
            if (j - i == 1) {
                bnd.push_back((int32_t)(edges[i] >> 32));
                bnd.push_back((int32_t)(edges[i] & 0xffffffffu));
            }
            i = j;
        }
        std::sort(bnd.begin(), bnd.end());
        bnd.erase(std::unique(bnd.begin(), bnd.end()), bnd.end());
    }
    // element_geometry (problems.hpp:115-128) validates every element
    for (long t = 0; t < ne; ++t) {
        const int32_t* v = &tri[3 * (size_t)t];
        const double x0 = xy[2 * (size_t)v[0]], y0 = xy[2 * (size_t)v[0] + 1];
        const double x1 = xy[2 * (size_t)v[1]], y1 = xy[2 * (size_t)v[1] + 1];
        const double x2 = xy[2 * (size_t)v[2]], y2 = xy[2 * (size_t)v[2] + 1];
        const double two_area = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0);
        if (!(std::abs(two_area) / 2.0 > 1e-14))
            throw AuxIoError(AUX_GEOMETRY_ERROR, "triangle " + std::to_string(t) + " is degenerate");
    }
    D->kind = 1;
    D->a = nn;
    D->b = ne;
    D->c = (int64_t)bnd.size();
    D->d0 = std::move(xy);
    D->i0 = std::move(tri);
    D->i1 = std::move(bnd);
}

void read_coords_file(const char* path, int threads, aux_file_data* D) {
    const std::vector<char> buf = slurp(path);
    const int T0 = pick_threads(threads);
    std::vector<std::vector<double>> pts(T0 + 1);
    std::vector<LineErr> err(T0 + 1);
    std::vector<long> lines;
    parallel_lines(buf.data(), buf.data() + buf.size(), T0, lines, [&](int t, const char* b, const char* e, long k) {
        if (err[t].line >= 0 || blank(b, e)) return;
        const char* p = b;
        double x = 0.0, y = 0.0;
        if (!get_double(p, e, x) || !get_double(p, e, y)) {
            err[t] = {k, "malformed coordinate line"};
            return;
        }
        pts[t].push_back(x);
        pts[t].push_back(y);
    });
    long base = 0;
    for (int t = 0; t < (int)lines.size(); ++t) {
        if (err[t].line >= 0) parse_fail(err[t].what, base + err[t].line + 1);
        base += lines[t];
    }
    D->kind = 2;
    for (int t = 0; t < (int)lines.size(); ++t) D->d0.insert(D->d0.end(), pts[t].begin(), pts[t].end());
    D->a = (int64_t)D->d0.size() / 2;
}

template <class F>
aux_status guarded(char* msg, size_t msg_len, F f) {
    auto put = [&](const char* s) {
        if (msg && msg_len) {
            std::strncpy(msg, s, msg_len - 1);
            msg[msg_len - 1] = '\0';
        }
    };
    try {
        f();
        put("");
        return AUX_OK;
    } catch (const AuxIoError& e) {
        put(e.what());
        return e.st;
    } catch (const std::bad_alloc&) {
        put("out of host memory");
        return AUX_CAPACITY_ERROR;
    } catch (const std::exception& e) {
        put(e.what());
        return AUX_INTERNAL_ERROR;
    }
}

}  // namespace

extern "C" {

aux_status aux_read_matrix_market(const char* path, int32_t threads, aux_file_data** out, char* msg, size_t msg_len) {
    *out = nullptr;
    auto* D = new aux_file_data();
    const aux_status st = guarded(msg, msg_len, [&] { read_mm(path, threads, D); });
    if (st != AUX_OK) delete D;
    else *out = D;
    return st;
}

aux_status aux_read_mesh(const char* path, int32_t threads, aux_file_data** out, char* msg, size_t msg_len) {
    *out = nullptr;
    auto* D = new aux_file_data();
    const aux_status st = guarded(msg, msg_len, [&] { read_mesh_file(path, threads, D); });
    if (st != AUX_OK) delete D;
    else *out = D;
    return st;
}

aux_status aux_read_coords(const char* path, int32_t threads, aux_file_data** out, char* msg, size_t msg_len) {
    *out = nullptr;
    auto* D = new aux_file_data();
    const aux_status st = guarded(msg, msg_len, [&] { read_coords_file(path, threads, D); });
    if (st != AUX_OK) delete D;
    else *out = D;
    return st;
}

aux_status aux_file_data_sizes(const aux_file_data* d, int64_t* a, int64_t* b, int64_t* c) {
    if (!d) return AUX_ARGUMENT_ERROR;
    if (a) *a = d->a;
    if (b) *b = d->b;
    if (c) *c = d->c;
    return AUX_OK;
}

aux_status aux_file_data_copy(const aux_file_data* d, void* p0, void* p1, void* p2) {
    if (!d) return AUX_ARGUMENT_ERROR;
    auto cp = [](void* dst, const void* src, size_t bytes) {
        if (dst && bytes) std::memcpy(dst, src, bytes);
    };
    if (d->kind == 0) {   // row_ptr, col_idx, values
        cp(p0, d->i0.data(), d->i0.size() * sizeof(int32_t));
        cp(p1, d->i1.data(), d->i1.size() * sizeof(int32_t));
        cp(p2, d->d0.data(), d->d0.size() * sizeof(double));
    } else if (d->kind == 1) {   // nodes xy, triangles, boundary nodes
        cp(p0, d->d0.data(), d->d0.size() * sizeof(double));
        cp(p1, d->i0.data(), d->i0.size() * sizeof(int32_t));
        cp(p2, d->i1.data(), d->i1.size() * sizeof(int32_t));
    } else {   // points xy
        cp(p0, d->d0.data(), d->d0.size() * sizeof(double));
    }
    return AUX_OK;
}

void aux_file_data_destroy(aux_file_data* d) { delete d; }

aux_status aux_write_matrix_market(const aux_csr_view* A, const char* path, char* msg, size_t msg_len) {
    return guarded(msg, msg_len, [&] {
        FILE* f = std::fopen(path, "wb");
        if (!f) io_fail(std::string("cannot open ") + path + " for writing");
        std::string out = "%%MatrixMarket matrix coordinate real general\n";
        out += std::to_string(A->n_rows) + " " + std::to_string(A->n_cols) + " " +
               std::to_string((long long)A->row_ptr[A->n_rows]) + "\n";
        char line[96];
        for (int r = 0; r < A->n_rows; ++r)
            for (int p = A->row_ptr[r]; p < A->row_ptr[r + 1]; ++p) {
                std::snprintf(line, sizeof line, "%d %d %.17g\n", r + 1, A->col_idx[p] + 1, A->values[p]);
                out += line;
            }
        const bool ok = std::fwrite(out.data(), 1, out.size(), f) == out.size();
        std::fclose(f);
        if (!ok) io_fail(std::string("write to ") + path + " failed");
    });
}

}  // extern "C"
