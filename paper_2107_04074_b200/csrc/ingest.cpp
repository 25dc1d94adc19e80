// ingest.cpp -- SVMlight/libsvm parsing and TF-IDF weights on the host
// (reference corpus_io.py:31-131), compiled into libspkm.so.
//
// The reference builds one Python SparseVector per line (its host-side
// scalability wall).  Here the file is parsed in
// parallel: the buffer is cut at line boundaries into one chunk per thread,
// every chunk is parsed into flat CSR pieces, and the pieces are joined in
// file order.  The grammar follows the reference exactly:
//   * universal newlines ('\n', '\r\n', lone '\r'); line numbers are 1-based
//     and count blank and comment lines;
//   * text after the first '#' is dropped, then Python str.strip()/split()
//     whitespace rules (ASCII: space, \t \n \v \f \r and \x1c-\x1f);
//   * a first token without ':' is a label and is discarded;
//   * pair = head ':' tail with Python int() / float() grammars (sign,
//     underscores between digits, inf / infinity / nan), converted with
//     strtod (correctly rounded, as CPython's float());
//   * indices must increase strictly (checked before explicit zeros are
//     dropped, corpus_io.py:68-72); errors carry the first failing line and
//     the reference's message text.
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "../../include/spkm.h"

namespace {

inline bool py_space(unsigned char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1f);
}
inline bool is_digit(char c) { return c >= '0' && c <= '9'; }

// Python repr() of an ASCII token (quote choice and escapes as CPython)
std::string py_repr(const char *b, const char *e) {
    bool has_sq = false, has_dq = false;
    for (const char *p = b; p < e; ++p) {
        has_sq |= *p == '\'';
        has_dq |= *p == '"';
    }
    const char q = (has_sq && !has_dq) ? '"' : '\'';
    std::string s(1, q);
    for (const char *p = b; p < e; ++p) {
        const unsigned char c = (unsigned char)*p;
        if (c == (unsigned char)q || c == '\\') {
            s += '\\';
            s += (char)c;
        } else if (c == '\t') {
            s += "\\t";
        } else if (c == '\n') {
            s += "\\n";
        } else if (c == '\r') {
            s += "\\r";
        } else if (c < 0x20 || c == 0x7f) {
            char buf[8];
            snprintf(buf, sizeof buf, "\\x%02x", c);
            s += buf;
        } else {
            s += (char)c;
        }
    }
    s += q;
    return s;
}

// digitpart := digit (["_"] digit)*; appends the digits to out
bool digitpart(const char *&p, const char *e, std::string &out) {
    if (p >= e || !is_digit(*p)) return false;
    while (p < e) {
        if (is_digit(*p)) {
            out += *p++;
        } else if (*p == '_' && p + 1 < e && is_digit(p[1]) && !out.empty()) {
            ++p;
        } else {
            break;
        }
    }
    return true;
}

// Python int(str) for base 10 (ASCII): [sign] digitpart
bool py_int(const char *b, const char *e, int64_t &v) {
    const char *p = b;
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) neg = (*p++ == '-');
    std::string d;
    if (!digitpart(p, e, d) || p != e) return false;
    unsigned long long acc = 0;
    for (char c : d) {
        const unsigned long long nx = acc * 10 + (unsigned long long)(c - '0');
        if (acc > (~0ull) / 10 || nx < acc) return false;   // beyond int64: not representable
        acc = nx;
    }
    if (!neg && acc > (unsigned long long)INT64_MAX) return false;
    if (neg && acc > (unsigned long long)INT64_MAX + 1ull) return false;
    v = neg ? (int64_t)(0 - acc) : (int64_t)acc;
    return true;
}

bool ieq(const char *b, const char *e, const char *word) {
    const size_t n = strlen(word);
    if ((size_t)(e - b) != n) return false;
    for (size_t i = 0; i < n; ++i)
        if (tolower((unsigned char)b[i]) != word[i]) return false;
    return true;
}

// Python float(str) grammar (ASCII), value by strtod on the cleaned text
bool py_float(const char *b, const char *e, double &v) {
    const char *p = b;
    std::string t;
    if (p < e && (*p == '+' || *p == '-')) t += *p++;
    if (ieq(p, e, "inf") || ieq(p, e, "infinity")) {
        v = (t == "-") ? -INFINITY : INFINITY;
        return true;
    }
    if (ieq(p, e, "nan")) {
        v = (t == "-") ? -NAN : NAN;
        return true;
    }
    bool mant = false;
    std::string d;
    if (p < e && is_digit(*p)) {
        if (!digitpart(p, e, d)) return false;
        t += d;
        mant = true;
    }
    if (p < e && *p == '.') {
        t += *p++;
        d.clear();
        if (p < e && is_digit(*p)) {
            if (!digitpart(p, e, d)) return false;
            t += d;
            mant = true;
        }
    }
    if (!mant) return false;
    if (p < e && (*p == 'e' || *p == 'E')) {
        t += *p++;
        if (p < e && (*p == '+' || *p == '-')) t += *p++;
        d.clear();
        if (!digitpart(p, e, d)) return false;
        t += d;
    }
    if (p != e) return false;
    v = strtod(t.c_str(), nullptr);
    return true;
}

struct Piece {
    std::vector<int64_t> row_nnz, idx;
    std::vector<double> val;
    int64_t max_idx = -1;
    int64_t err_line = 0;
    std::string err_msg;
};

// parse [b, e) whose first line is line number `line0`
void parse_chunk(const char *b, const char *e, int64_t line0, Piece &out) {
    int64_t line = line0;
    const char *p = b;
    std::vector<const char *> tb, te;
    std::vector<int64_t> ri;
    std::vector<double> rv;
    while (p < e) {
        const char *ls = p;
        while (p < e && *p != '\n' && *p != '\r') ++p;
        const char *le = p;
        if (p < e) {
            if (*p == '\r' && p + 1 < e && p[1] == '\n') p += 2;
            else ++p;
        }
        const char *hash = (const char *)memchr(ls, '#', (size_t)(le - ls));
        if (hash) le = hash;
        tb.clear();
        te.clear();
        for (const char *q = ls; q < le;) {
            while (q < le && py_space((unsigned char)*q)) ++q;
            if (q >= le) break;
            const char *s0 = q;
            while (q < le && !py_space((unsigned char)*q)) ++q;
            tb.push_back(s0);
            te.push_back(q);
        }
        if (tb.empty()) {
            ++line;
            continue;
        }
        size_t first = memchr(tb[0], ':', (size_t)(te[0] - tb[0])) ? 0 : 1;   // label, discarded
        ri.clear();
        rv.clear();
        int64_t prev = -1;
        for (size_t t = first; t < tb.size(); ++t) {
            const char *c = (const char *)memchr(tb[t], ':', (size_t)(te[t] - tb[t]));
            if (!c) {
                out.err_line = line;
                out.err_msg = "malformed pair " + py_repr(tb[t], te[t]);
                return;
            }
            int64_t i;
            double v;
            if (!py_int(tb[t], c, i) || !py_float(c + 1, te[t], v)) {
                out.err_line = line;
                out.err_msg = "non-numeric pair " + py_repr(tb[t], te[t]);
                return;
            }
            if (i <= prev) {
                out.err_line = line;
                out.err_msg = "indices not strictly increasing at " + py_repr(tb[t], te[t]);
                return;
            }
            prev = i;
            ri.push_back(i);
            rv.push_back(v);
        }
        int64_t kept = 0;
        for (size_t q = 0; q < ri.size(); ++q) {
            if (rv[q] != 0.0) {   // explicit zeros are dropped (sparse.py:34-36)
                out.idx.push_back(ri[q]);
                out.val.push_back(rv[q]);
                ++kept;
                out.max_idx = std::max(out.max_idx, ri[q]);
            }
        }
        out.row_nnz.push_back(kept);
        ++line;
    }
}

int64_t count_lines(const char *b, const char *e) {
    int64_t n = 0;
    for (const char *p = b; p < e; ++p) {
        if (*p == '\n') ++n;
        else if (*p == '\r' && !(p + 1 < e && p[1] == '\n')) ++n;
    }
    return n;
}

struct Parsed {
    std::vector<Piece> pieces;
};

}  // namespace

extern "C" {

int spkm_svml_parse(const char *buf, int64_t len, int nthreads, spkm_svml *out) {
    memset(out, 0, sizeof *out);
    if (nthreads < 1) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
    if (nthreads > 64) nthreads = 64;
    if (len < (int64_t)1 << 20) nthreads = 1;
    // chunk boundaries right after a '\n'
    std::vector<const char *> cut{buf};
    for (int t = 1; t < nthreads; ++t) {
        const char *p = buf + len * t / nthreads;
        if (p <= cut.back()) continue;
        const char *nl = (const char *)memchr(p, '\n', (size_t)(buf + len - p));
        if (!nl) break;
        if (nl + 1 > cut.back() && nl + 1 < buf + len) cut.push_back(nl + 1);
    }
    cut.push_back(buf + len);
    const size_t nc = cut.size() - 1;
    std::vector<int64_t> line0(nc, 1);
    {
        std::vector<int64_t> cnt(nc, 0);
        std::vector<std::thread> th;
        for (size_t c = 0; c < nc; ++c) th.emplace_back([&, c] { cnt[c] = count_lines(cut[c], cut[c + 1]); });
        for (auto &x : th) x.join();
        for (size_t c = 1; c < nc; ++c) line0[c] = line0[c - 1] + cnt[c - 1];
    }
    Parsed *P = new Parsed();
    P->pieces.resize(nc);
    {
        std::vector<std::thread> th;
        for (size_t c = 0; c < nc; ++c)
            th.emplace_back([&, c] { parse_chunk(cut[c], cut[c + 1], line0[c], P->pieces[c]); });
        for (auto &x : th) x.join();
    }
    out->max_idx = -1;
    for (size_t c = 0; c < nc; ++c) {
        const Piece &pc = P->pieces[c];
        if (pc.err_line) {
            out->err_line = pc.err_line;
            snprintf(out->err_msg, sizeof out->err_msg, "%s", pc.err_msg.c_str());
            delete P;
            return 1;
        }
        out->n_rows += (int64_t)pc.row_nnz.size();
        out->nnz += (int64_t)pc.idx.size();
        out->max_idx = std::max(out->max_idx, pc.max_idx);
    }
    out->handle = P;
    return 0;
}

int spkm_svml_fetch(spkm_svml *res, int64_t *indptr, int64_t *indices, double *values) {
    Parsed *P = static_cast<Parsed *>(res->handle);
    if (!P) return -1;
    int64_t r = 0, z = 0;
    indptr[0] = 0;
    for (const Piece &pc : P->pieces) {
        for (int64_t m : pc.row_nnz) {
            indptr[r + 1] = indptr[r] + m;
            ++r;
        }
        if (!pc.idx.empty()) {
            memcpy(indices + z, pc.idx.data(), sizeof(int64_t) * pc.idx.size());
            memcpy(values + z, pc.val.data(), sizeof(double) * pc.val.size());
        }
        z += (int64_t)pc.idx.size();
    }
    delete P;
    res->handle = nullptr;
    return 0;
}

int spkm_svml_free(spkm_svml *res) {
    delete static_cast<Parsed *>(res->handle);
    res->handle = nullptr;
    return 0;
}

// idf of every term with df > 0 (corpus_io.py:104-107): ln(n / df), or
// ln((1 + n) / (1 + df)) + 1 when smooth; libm log as CPython's math.log.
int spkm_host_idf(int64_t d, const int64_t *df, int64_t n, int smooth, double *idf) {
    for (int64_t j = 0; j < d; ++j) {
        if (df[j] <= 0) {
            idf[j] = 0.0;
            continue;
        }
        idf[j] = smooth ? log((1.0 + (double)n) / (1.0 + (double)df[j])) + 1.0 : log((double)n / (double)df[j]);
    }
    return 0;
}

}  // extern "C"
