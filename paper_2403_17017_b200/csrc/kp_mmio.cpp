// kp_mmio.cpp -- Matrix Market coordinate ingest (sparse.py:106-196), native and parallel.
//
// The wire format in front of csr_from_coo.  Restates the reference's
// parse_matrix_market line by line: Python `str.splitlines()` line breaks (\n, \r, \r\n,
// \v, \f, \x1c-\x1e, U+0085, U+2028, U+2029) for the 1-based line numbers in errors, the
// `strip()` / `split()` whitespace, the header / size-line / entry checks in the same
// order and with the same messages, int() / float() token grammar (sign, digits with
// single underscores, inf / infinity / nan; no hex), symmetric mirroring appended right
// after each entry.  Float conversion is glibc strtod on the underscore-free token:
// correctly rounded, i.e. identical to Python's float() for every decimal literal.
//
// Parallel: the buffer is split into per-thread chunks at line starts; pass 1 counts line
// breaks and entry lines per chunk, pass 2 parses each chunk with its global line number
// and entry index (so "extra data" and every error report the same first line the
// sequential reference reports), pass 3 concatenates the per-chunk triples in order.
// Out of scope (documented divergence): non-ASCII digits / whitespace, which Python's
// int()/float()/split() would accept.
#include <errno.h>
#include <omp.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/kernelpick_b200.h"

namespace {

// ---- Python splitlines() break at p (returns break length, 0 if none)
inline size_t brk(const char *p, const char *e) {
    const unsigned char c = (unsigned char)*p;
    if (c == '\n' || c == '\v' || c == '\f' || c == 0x1c || c == 0x1d || c == 0x1e) return 1;
    if (c == '\r') return (p + 1 < e && p[1] == '\n') ? 2 : 1;
    if (c == 0xc2 && p + 1 < e && (unsigned char)p[1] == 0x85) return 2;  // U+0085
    if (c == 0xe2 && p + 2 < e && (unsigned char)p[1] == 0x80 &&
        ((unsigned char)p[2] == 0xa8 || (unsigned char)p[2] == 0xa9))
        return 3;  // U+2028 / U+2029
    return 0;
}
inline bool ws(char c) { return c == ' ' || c == '\t' || c == 0x1f; }

struct Line {
    const char *b, *e;  // stripped
};
inline Line strip(const char *b, const char *e) {
    while (b < e && ws(*b)) ++b;
    while (e > b && ws(e[-1])) --e;
    return {b, e};
}
inline int split(Line l, Line *tok, int max_tok) {
    int n = 0;
    const char *p = l.b;
    while (p < l.e) {
        while (p < l.e && ws(*p)) ++p;
        if (p >= l.e) break;
        const char *s = p;
        while (p < l.e && !ws(*p)) ++p;
        if (n < max_tok) tok[n] = {s, p};
        ++n;
    }
    return n;
}

// Python int(): [+-]? digit ( _? digit )*  (ASCII); saturates on overflow (out of range anyway)
bool py_int(Line t, int64_t *out, bool *overflow) {
    const char *p = t.b;
    bool neg = false;
    if (p < t.e && (*p == '+' || *p == '-')) neg = *p++ == '-';
    if (p >= t.e || *p < '0' || *p > '9') return false;
    unsigned __int128 v = 0;
    bool ovf = false, prev_us = false;
    for (; p < t.e; ++p) {
        if (*p == '_') {
            if (prev_us || p + 1 >= t.e) return false;
            prev_us = true;
            continue;
        }
        if (*p < '0' || *p > '9') return false;
        prev_us = false;
        v = v * 10 + (unsigned)(*p - '0');
        if (v > ((unsigned __int128)1 << 64)) { ovf = true; v = (unsigned __int128)1 << 64; }
    }
    if (v > (unsigned __int128)INT64_MAX) ovf = true;
    *overflow = ovf;
    *out = ovf ? (neg ? INT64_MIN : INT64_MAX) : (neg ? -(int64_t)v : (int64_t)v);
    return true;
}

// Python float(): decimal literal with optional single underscores between digits, or
// inf / infinity / nan (any case, optional sign).  Returns false when Python would raise.
bool py_float(Line t, double *out) {
    const char *p = t.b;
    const size_t n = (size_t)(t.e - t.b);
    if (n == 0 || n > 512) return n != 0 && false;
    char buf[520];
    size_t k = 0;
    const char *q = p;
    if (*q == '+' || *q == '-') buf[k++] = *q++;
    // specials
    {
        char low[16];
        size_t m = (size_t)(t.e - q);
        if (m <= 8) {
            for (size_t i = 0; i < m; ++i) low[i] = (char)((q[i] >= 'A' && q[i] <= 'Z') ? q[i] + 32 : q[i]);
            low[m] = 0;
            if (!strcmp(low, "inf") || !strcmp(low, "infinity")) {
                *out = (buf[0] == '-' && k) ? -INFINITY : INFINITY;
                return true;
            }
            if (!strcmp(low, "nan")) {
                *out = NAN;
                return true;
            }
        }
    }
    // grammar: digitpart? ('.' digitpart?)? (e [+-]? digitpart)? with at least one digit in mantissa
    auto digitpart = [&](const char *&s) -> int {  // returns digits copied, -1 on bad underscore
        int d = 0;
        bool prev_digit = false;
        while (s < t.e) {
            if (*s >= '0' && *s <= '9') {
                buf[k++] = *s++;
                ++d;
                prev_digit = true;
            } else if (*s == '_') {
                if (!prev_digit || s + 1 >= t.e || s[1] < '0' || s[1] > '9') return -1;
                ++s;
                prev_digit = false;
            } else {
                break;
            }
        }
        return d;
    };
    int d1 = digitpart(q);
    if (d1 < 0) return false;
    int d2 = 0;
    if (q < t.e && *q == '.') {
        buf[k++] = *q++;
        d2 = digitpart(q);
        if (d2 < 0) return false;
    }
    if (d1 + d2 == 0) return false;
    if (q < t.e && (*q == 'e' || *q == 'E')) {
        buf[k++] = *q++;
        if (q < t.e && (*q == '+' || *q == '-')) buf[k++] = *q++;
        const int d3 = digitpart(q);
        if (d3 <= 0) return false;
    }
    if (q != t.e) return false;
    buf[k] = 0;
    errno = 0;
    char *endp = nullptr;
    *out = strtod(buf, &endp);  // correctly rounded (glibc); ERANGE over/underflow = inf / 0 like Python
    return endp == buf + k;
}

void set_err(kp_mm_info *info, int64_t line, const std::string &msg) {
    info->err_line = line;
    snprintf(info->err, sizeof(info->err), "%s", msg.c_str());
}

std::string quote(Line l) {  // Python repr() of an ASCII str (single quotes unless it contains ')
    std::string s(l.b, l.e);
    const bool dq = s.find('\'') != std::string::npos && s.find('"') == std::string::npos;
    std::string r(1, dq ? '"' : '\'');
    for (unsigned char c : s) {
        if (c == '\\') r += "\\\\";
        else if (!dq && c == '\'') r += "\\'";
        else if (c == '\t') r += "\\t";
        else if (c < 0x20 || c == 0x7f) {
            char h[8];
            snprintf(h, sizeof(h), "\\x%02x", c);
            r += h;
        } else r += (char)c;
    }
    r += dq ? '"' : '\'';
    return r;
}

struct Header {
    int64_t n_rows = 0, n_cols = 0, n_entries = 0;
    int pattern = 0, symmetry = 0;  // 0 general, 1 symmetric, 2 skew
    int field = 0;
    const char *entries = nullptr;  // first byte after the size line's break
    int64_t next_line = 0;          // line number of the first line after the size line
};

// header + size line (sequential, sparse.py:114-152)
int parse_header(const char *buf, size_t len, Header *H, kp_mm_info *info) {
    const char *e = buf + len;
    // line 1
    const char *p = buf;
    while (p < e && !brk(p, e)) ++p;
    if (len == 0) {
        set_err(info, 1, "line 1: empty file, missing Matrix Market header");
        return KP_EPARSE;
    }
    Line h = strip(buf, p);
    std::string low(h.b, h.e);
    for (auto &c : low) c = (char)((c >= 'A' && c <= 'Z') ? c + 32 : c);
    Line lowl{low.data(), low.data() + low.size()};
    Line tk[6];
    const int nt = split(lowl, tk, 6);
    if (nt != 5 || std::string(tk[0].b, tk[0].e) != "%%matrixmarket") {
        set_err(info, 1, "line 1: malformed header " + quote(h));
        return KP_EPARSE;
    }
    const std::string obj(tk[1].b, tk[1].e), fmt(tk[2].b, tk[2].e), field(tk[3].b, tk[3].e), sym(tk[4].b, tk[4].e);
    if (obj != "matrix") { set_err(info, 1, "line 1: unsupported object " + quote(tk[1])); return KP_EPARSE; }
    if (fmt != "coordinate") {
        set_err(info, 1, "line 1: unsupported format " + quote(tk[2]) + " (coordinate only)");
        return KP_EPARSE;
    }
    if (field == "real") H->field = 0;
    else if (field == "integer") H->field = 1;
    else if (field == "pattern") H->field = 2;
    else {
        set_err(info, 1, "line 1: unsupported field " + quote(tk[3]) + " (complex data is out of scope)");
        return KP_EPARSE;
    }
    if (sym == "general") H->symmetry = 0;
    else if (sym == "symmetric") H->symmetry = 1;
    else if (sym == "skew-symmetric") H->symmetry = 2;
    else { set_err(info, 1, "line 1: unsupported symmetry " + quote(tk[4])); return KP_EPARSE; }
    H->pattern = H->field == 2;
    // size line
    int64_t lineno = 1;
    p += p < e ? brk(p, e) : 0;
    bool got = false;
    while (p < e) {
        const char *s = p;
        while (p < e && !brk(p, e)) ++p;
        ++lineno;
        Line l = strip(s, p);
        p += p < e ? brk(p, e) : 0;
        if (l.b == l.e || *l.b == '%') continue;
        Line t[4];
        const int n = split(l, t, 4);
        char msg[64];
        snprintf(msg, sizeof(msg), "line %lld: ", (long long)lineno);
        if (n != 3) {
            set_err(info, lineno, std::string(msg) + "size line must be 'rows cols nnz', got " + quote(l));
            return KP_EPARSE;
        }
        int64_t v[3];
        for (int i = 0; i < 3; ++i) {
            bool ovf = false;
            if (!py_int(t[i], &v[i], &ovf) || ovf) {
                set_err(info, lineno, std::string(msg) + "non-integer size line " + quote(l));
                return KP_EPARSE;
            }
        }
        if (v[0] < 0 || v[1] < 0 || v[2] < 0) {
            set_err(info, lineno, std::string(msg) + "negative size values");
            return KP_EPARSE;
        }
        H->n_rows = v[0]; H->n_cols = v[1]; H->n_entries = v[2];
        got = true;
        break;
    }
    if (!got) {
        char msg[64];
        snprintf(msg, sizeof(msg), "line %lld: missing size line", (long long)lineno);
        set_err(info, lineno, msg);
        return KP_EPARSE;
    }
    H->entries = p;
    H->next_line = lineno + 1;
    info->n_rows = H->n_rows; info->n_cols = H->n_cols; info->n_entries = H->n_entries;
    info->field = H->field; info->symmetry = H->symmetry;
    return KP_OK;
}

struct Chunk {
    const char *b, *e;
    int64_t lines = 0, entries = 0;       // pass 1
    int64_t line0 = 0, entry0 = 0;        // global numbering of the chunk's first line / entry
    std::vector<int64_t> r, c;
    std::vector<double> v;
    int64_t err_line = INT64_MAX;
    std::string err;
    bool ends_with_break = false;
};

}  // namespace

extern "C" {

int kp_mm_header(const char *buf, size_t len, kp_mm_info *info) {
    if (!info || (len && !buf)) return KP_EINVAL;
    memset(info, 0, sizeof(*info));
    Header H;
    return parse_header(buf, len, &H, info);
}

int kp_mm_parse(const char *buf, size_t len, int64_t *rows, int64_t *cols, double *vals, int64_t capacity,
                int32_t n_threads, kp_mm_info *info) {
    if (!info || (len && !buf) || capacity < 0) return KP_EINVAL;
    memset(info, 0, sizeof(*info));
    Header H;
    int rc = parse_header(buf, len, &H, info);
    if (rc) return rc;
    const char *e = buf + len;
    const char *s0 = H.entries;
    int T = n_threads > 0 ? n_threads : omp_get_max_threads();
    const size_t body = (size_t)(e - s0);
    if (body < (size_t)T * 4096) T = std::max<int>(1, (int)(body / 4096));
    // chunk boundaries at line starts
    std::vector<Chunk> ch(T);
    {
        std::vector<const char *> cut(T + 1);
        cut[0] = s0;
        cut[T] = e;
        for (int t = 1; t < T; ++t) {
            const char *p = s0 + body * (size_t)t / (size_t)T;
            if (p < cut[t - 1]) p = cut[t - 1];
            // advance to the first byte after a line break
            while (p < e) {
                const size_t b = brk(p, e);
                if (b) {
                    // \r\n must not be split, nor multi-byte breaks (p is their first byte here)
                    if (p > s0 && *p == '\n' && p[-1] == '\r') { p += 1; break; }
                    p += b;
                    break;
                }
                ++p;
            }
            cut[t] = p;
        }
        for (int t = 0; t < T; ++t) {
            ch[t].b = cut[t];
            ch[t].e = std::max(cut[t], cut[t + 1]);
        }
    }
    const bool pattern = H.pattern;
    const int want = pattern ? 2 : 3;
    // pass 1: lines and entry lines per chunk
#pragma omp parallel for num_threads(T) schedule(static, 1)
    for (int t = 0; t < T; ++t) {
        Chunk &c = ch[t];
        const char *p = c.b;
        while (p < c.e) {
            const char *s = p;
            while (p < c.e && !brk(p, c.e)) ++p;
            Line l = strip(s, p);
            ++c.lines;
            if (l.b != l.e && *l.b != '%') ++c.entries;
            if (p < c.e) p += brk(p, c.e);
        }
    }
    int64_t ln = H.next_line, en = 0;
    for (int t = 0; t < T; ++t) {
        ch[t].line0 = ln;
        ch[t].entry0 = en;
        ln += ch[t].lines;
        en += ch[t].entries;
    }
    // pass 2: parse
#pragma omp parallel for num_threads(T) schedule(static, 1)
    for (int t = 0; t < T; ++t) {
        Chunk &c = ch[t];
        c.r.reserve((size_t)c.entries * (H.symmetry ? 2 : 1));
        c.c.reserve((size_t)c.entries * (H.symmetry ? 2 : 1));
        c.v.reserve((size_t)c.entries * (H.symmetry ? 2 : 1));
        const char *p = c.b;
        int64_t lineno = c.line0, seen = c.entry0;
        char pre[48];
        while (p < c.e) {
            const char *s = p;
            while (p < c.e && !brk(p, c.e)) ++p;
            Line l = strip(s, p);
            if (p < c.e) p += brk(p, c.e);
            const int64_t this_line = lineno++;
            if (l.b == l.e || *l.b == '%') continue;
            snprintf(pre, sizeof(pre), "line %lld: ", (long long)this_line);
            if (seen == H.n_entries) {
                c.err_line = this_line;
                c.err = std::string(pre) + "extra data after " + std::to_string(H.n_entries) + " entries";
                break;
            }
            Line tk[4];
            const int nt = split(l, tk, 4);
            if (nt != want) {
                c.err_line = this_line;
                c.err = std::string(pre) + "expected " + std::to_string(want) + " fields, got " + std::to_string(nt);
                break;
            }
            int64_t i, j;
            bool oi = false, oj = false;
            double v = 1.0;
            if (!py_int(tk[0], &i, &oi) || !py_int(tk[1], &j, &oj) || (!pattern && !py_float(tk[2], &v))) {
                c.err_line = this_line;
                c.err = std::string(pre) + "malformed entry " + quote(l);
                break;
            }
            if (!std::isfinite(v)) {
                c.err_line = this_line;
                c.err = std::string(pre) + "non-finite value " + quote(tk[nt - 1]);
                break;
            }
            if (oi || oj || !(1 <= i && i <= H.n_rows) || !(1 <= j && j <= H.n_cols)) {
                c.err_line = this_line;
                c.err = std::string(pre) + "index (" + std::string(tk[0].b, tk[0].e) + ", " +
                        std::string(tk[1].b, tk[1].e) + ") out of range";
                if (!oi && !oj) c.err = std::string(pre) + "index (" + std::to_string(i) + ", " + std::to_string(j) + ") out of range";
                break;
            }
            if (H.symmetry == 2 && i == j) {
                c.err_line = this_line;
                c.err = std::string(pre) + "diagonal entry in skew-symmetric file";
                break;
            }
            c.r.push_back(i - 1);
            c.c.push_back(j - 1);
            c.v.push_back(v);
            if (H.symmetry != 0 && i != j) {
                c.r.push_back(j - 1);
                c.c.push_back(i - 1);
                c.v.push_back(H.symmetry == 2 ? -v : v);
            }
            ++seen;
        }
    }
    // first error in line order == the sequential reference's error
    int64_t best = INT64_MAX;
    const Chunk *bc = nullptr;
    for (auto &c : ch)
        if (c.err_line < best) { best = c.err_line; bc = &c; }
    if (bc) {
        set_err(info, best, bc->err);
        return KP_EPARSE;
    }
    if (en != H.n_entries) {
        // reference: "line {len(lines)}: truncated ..." -- len(splitlines()) counts lines
        const int64_t nlines = H.next_line - 1 + (ln - H.next_line);
        char msg[160];
        snprintf(msg, sizeof(msg), "line %lld: truncated entry list, expected %lld entries, got %lld",
                 (long long)nlines, (long long)H.n_entries, (long long)en);
        set_err(info, nlines, msg);
        return KP_EPARSE;
    }
    int64_t total = 0;
    for (auto &c : ch) total += (int64_t)c.r.size();
    info->n_triples = total;
    if (total > capacity || (total && (!rows || !cols || !vals))) return KP_ENOMEM;
    std::vector<int64_t> at(T + 1, 0);
    for (int t = 0; t < T; ++t) at[t + 1] = at[t] + (int64_t)ch[t].r.size();
#pragma omp parallel for num_threads(T) schedule(static, 1)
    for (int t = 0; t < T; ++t) {
        const size_t m = ch[t].r.size();
        if (!m) continue;
        memcpy(rows + at[t], ch[t].r.data(), m * sizeof(int64_t));
        memcpy(cols + at[t], ch[t].c.data(), m * sizeof(int64_t));
        memcpy(vals + at[t], ch[t].v.data(), m * sizeof(double));
    }
    return KP_OK;
}

}  // extern "C"
