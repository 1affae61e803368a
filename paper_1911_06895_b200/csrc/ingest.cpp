// ingest.cpp -- native graph-file parsing behind ds_ingest_* (include/dsssp.h).
//
// Restates the reference loaders (deltasparse/io.py) over an in-memory byte
// buffer: Matrix Market coordinate files (load_matrix_market, io.py:121-193)
// and whitespace edge lists (load_edge_list, io.py:196-259).  Same accepted
// grammar, same line numbering (universal newlines, 1-based, comment lines
// counted), same error texts and the same split between structural errors
// (DS_EPARSE -> ParseError) and unusable content (DS_EVALID ->
// ValidationError).  The output is the COO entry list in file order
// (symmetric / undirected inputs already mirrored, self-loops dropped and
// counted) plus, for edge lists, the first-seen label order; the caller
// builds the CSR with matrix_build semantics (duplicates keep the minimum).
#include <cerrno>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/dsssp.h"

extern int ds_internal_set_err(int code, const char* msg);

struct ds_ingest {
    int64_t n = 0;
    int64_t self_loops = 0;
    std::vector<int64_t> rows, cols;
    std::vector<double> vals;
    std::vector<int64_t> labels;  // external label of each internal id
};

namespace {

thread_local int64_t g_err_line = 0;

int fail(int code, const std::string& path, int64_t lineno, const char* fmt, ...) {
    char msg[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(msg, sizeof(msg), fmt, ap);
    va_end(ap);
    g_err_line = lineno;
    const std::string full = path + ":" + std::to_string(lineno) + ": " + msg;
    return ds_internal_set_err(code, full.c_str());
}

// str.split() / str.strip() whitespace (ASCII part: \t\n\v\f\r, \x1c-\x1f, space)
inline bool is_ws(unsigned char c) { return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f); }

struct Line {
    const char* p;
    size_t len;
};

// universal-newline line iterator (\n, \r\n, \r), like open(path, "r")
class Lines {
  public:
    Lines(const char* d, size_t n) : d_(d), n_(n) {}
    bool next(Line& l, int64_t& no) {
        if (pos_ >= n_) return false;
        const size_t s = pos_;
        while (pos_ < n_ && d_[pos_] != '\n' && d_[pos_] != '\r') ++pos_;
        l.p = d_ + s;
        l.len = pos_ - s;
        if (pos_ < n_) {
            if (d_[pos_] == '\r' && pos_ + 1 < n_ && d_[pos_ + 1] == '\n') ++pos_;
            ++pos_;
        }
        no = ++line_;
        return true;
    }

  private:
    const char* d_;
    size_t n_;
    size_t pos_ = 0;
    int64_t line_ = 0;
};

void split(const Line& l, std::vector<std::string>& out) {
    out.clear();
    size_t i = 0;
    while (i < l.len) {
        while (i < l.len && is_ws((unsigned char)l.p[i])) ++i;
        if (i >= l.len) break;
        const size_t s = i;
        while (i < l.len && !is_ws((unsigned char)l.p[i])) ++i;
        out.emplace_back(l.p + s, i - s);
    }
}

// int(token): optional sign, decimal digits with single underscores between
// digits (Python's integer literal rules for int(str))
bool parse_int(const std::string& t, int64_t& v) {
    size_t i = 0;
    bool neg = false;
    if (i < t.size() && (t[i] == '+' || t[i] == '-')) neg = t[i++] == '-';
    if (i >= t.size()) return false;
    unsigned long long acc = 0;
    bool prev_digit = false, any = false;
    for (; i < t.size(); ++i) {
        const char c = t[i];
        if (c >= '0' && c <= '9') {
            const unsigned long long nx = acc * 10 + (unsigned long long)(c - '0');
            if (nx / 10 != acc || nx > (unsigned long long)INT64_MAX + (neg ? 1 : 0)) return false;
            acc = nx;
            prev_digit = any = true;
        } else if (c == '_' && prev_digit && i + 1 < t.size()) {
            prev_digit = false;
        } else {
            return false;
        }
    }
    if (!any || !prev_digit) return false;
    v = neg ? (int64_t)(0 - acc) : (int64_t)acc;
    return true;
}

// float(token): decimal / exponent forms, inf / infinity / nan (any case),
// underscores between digits; hexadecimal floats are rejected like Python
bool parse_float(const std::string& t, double& v) {
    std::string s;
    s.reserve(t.size());
    for (size_t i = 0; i < t.size(); ++i) {
        if (t[i] == '_') {
            const bool ok = i > 0 && i + 1 < t.size() && isdigit((unsigned char)t[i - 1]) &&
                            isdigit((unsigned char)t[i + 1]);
            if (!ok) return false;
            continue;
        }
        s.push_back(t[i]);
    }
    if (s.empty()) return false;
    size_t k = (s[0] == '+' || s[0] == '-') ? 1 : 0;
    if (s.size() > k + 1 && s[k] == '0' && (s[k + 1] == 'x' || s[k + 1] == 'X')) return false;
    std::string low;
    for (char c : s.substr(k)) low.push_back((char)tolower((unsigned char)c));
    if (low == "inf" || low == "infinity") {
        v = (s[0] == '-') ? -INFINITY : INFINITY;
        return true;
    }
    if (low == "nan") {
        v = NAN;
        return true;
    }
    for (char c : low)
        if (!(isdigit((unsigned char)c) || c == '.' || c == 'e' || c == '+' || c == '-')) return false;
    errno = 0;
    char* end = nullptr;
    v = strtod(s.c_str(), &end);
    if (end != s.c_str() + s.size()) return false;
    return true;  // overflow gives +-inf, as float() does
}

int parse_weight(const std::string& tok, const std::string& path, int64_t lineno, double& w) {
    if (!parse_float(tok, w)) return fail(DS_EPARSE, path, lineno, "bad weight '%s'", tok.c_str());
    if (!(w > 0 && std::isfinite(w)))
        return fail(DS_EVALID, path, lineno, "edge weight must be strictly positive, got %s", tok.c_str());
    return DS_OK;
}

std::string lower(std::string s) {
    for (char& c : s) c = (char)tolower((unsigned char)c);
    return s;
}

Line strip(const Line& l) {
    size_t a = 0, b = l.len;
    while (a < b && is_ws((unsigned char)l.p[a])) ++a;
    while (b > a && is_ws((unsigned char)l.p[b - 1])) --b;
    return Line{l.p + a, b - a};
}

int parse_mtx(const char* data, size_t len, double default_weight, const std::string& path,
              ds_ingest* g) {
    Lines it(data, len);
    Line first;
    int64_t lineno = 0;
    if (!it.next(first, lineno)) return fail(DS_EPARSE, path, 1, "empty file");
    std::vector<std::string> tok;
    split(first, tok);
    for (auto& t : tok) t = lower(t);
    if (tok.size() != 5 || tok[0] != "%%matrixmarket")
        return fail(DS_EPARSE, path, lineno, "expected '%%%%MatrixMarket matrix coordinate ...' header");
    const std::string obj = tok[1], fmt = tok[2], field = tok[3], sym = tok[4];
    if (obj != "matrix" || fmt != "coordinate")
        return fail(DS_EPARSE, path, lineno, "unsupported layout '%s'/'%s'", obj.c_str(), fmt.c_str());
    if (field != "real" && field != "integer" && field != "pattern")
        return fail(DS_EPARSE, path, lineno, "unsupported field '%s'", field.c_str());
    if (sym != "general" && sym != "symmetric")
        return fail(DS_EPARSE, path, lineno, "unsupported symmetry '%s'", sym.c_str());
    const bool symmetric = sym == "symmetric";
    const size_t want = field == "pattern" ? 2 : 3;
    int64_t n = -1, declared = 0, seen = 0, last = lineno;
    Line raw;
    while (it.next(raw, lineno)) {
        last = lineno;
        const Line l = strip(raw);
        if (l.len == 0 || l.p[0] == '%') continue;
        split(l, tok);
        if (n < 0) {
            if (tok.size() != 3) return fail(DS_EPARSE, path, lineno, "expected 'rows cols entries' size line");
            int64_t nr, nc, d;
            if (!parse_int(tok[0], nr) || !parse_int(tok[1], nc) || !parse_int(tok[2], d))
                return fail(DS_EPARSE, path, lineno, "size line must hold three integers");
            if (nr != nc)
                return fail(DS_EPARSE, path, lineno, "graph matrix must be square, got %lldx%lld",
                            (long long)nr, (long long)nc);
            if (nr < 1) return fail(DS_EPARSE, path, lineno, "matrix dimension must be positive");
            n = nr;
            declared = d;
            if (declared > 0) {
                const size_t cap = (size_t)std::min<int64_t>(declared, 1 << 26) * (symmetric ? 2 : 1);
                g->rows.reserve(cap);
                g->cols.reserve(cap);
                g->vals.reserve(cap);
            }
            continue;
        }
        if (seen == declared)
            return fail(DS_EPARSE, path, lineno, "more than the declared %lld entries", (long long)declared);
        if (tok.size() != want)
            return fail(DS_EPARSE, path, lineno, "expected %zu tokens, got %zu", want, tok.size());
        int64_t r, c;
        if (!parse_int(tok[0], r) || !parse_int(tok[1], c))
            return fail(DS_EPARSE, path, lineno, "coordinates must be integers");
        if (!(1 <= r && r <= n && 1 <= c && c <= n))
            return fail(DS_EPARSE, path, lineno, "coordinate (%lld, %lld) outside 1..%lld", (long long)r,
                        (long long)c, (long long)n);
        double w = default_weight;
        if (field != "pattern") {
            const int rc = parse_weight(tok[2], path, lineno, w);
            if (rc) return rc;
        }
        ++seen;
        if (r == c) {
            ++g->self_loops;
            continue;
        }
        g->rows.push_back(r - 1);
        g->cols.push_back(c - 1);
        g->vals.push_back(w);
        if (symmetric) {
            g->rows.push_back(c - 1);
            g->cols.push_back(r - 1);
            g->vals.push_back(w);
        }
    }
    if (n < 0) return fail(DS_EPARSE, path, last, "missing size line");
    if (seen != declared)
        return fail(DS_EPARSE, path, last, "file ended after %lld of %lld entries", (long long)seen,
                    (long long)declared);
    g->n = n;
    g->labels.resize((size_t)n);
    for (int64_t i = 0; i < n; ++i) g->labels[(size_t)i] = i + 1;  // the file's 1-based numbers
    return DS_OK;
}

int parse_edges(const char* data, size_t len, bool directed, double default_weight,
                const std::string& path, ds_ingest* g) {
    Lines it(data, len);
    std::unordered_map<int64_t, int64_t> to_internal;
    auto intern = [&](int64_t label) -> int64_t {
        auto f = to_internal.find(label);
        if (f != to_internal.end()) return f->second;
        const int64_t id = (int64_t)g->labels.size();
        to_internal.emplace(label, id);
        g->labels.push_back(label);
        return id;
    };
    std::vector<std::string> tok;
    Line raw;
    int64_t lineno = 0, last = 0;
    while (it.next(raw, lineno)) {
        last = lineno;
        const Line l = strip(raw);
        if (l.len == 0 || l.p[0] == '#' || l.p[0] == '%') continue;
        split(l, tok);
        if (tok.size() != 2 && tok.size() != 3)
            return fail(DS_EPARSE, path, lineno, "expected 'u v' or 'u v w', got %zu tokens", tok.size());
        int64_t u, v;
        if (!parse_int(tok[0], u) || !parse_int(tok[1], v))
            return fail(DS_EPARSE, path, lineno, "vertex labels must be integers");
        if (u < 0 || v < 0) return fail(DS_EPARSE, path, lineno, "vertex labels must be non-negative");
        double w = default_weight;
        if (tok.size() == 3) {
            const int rc = parse_weight(tok[2], path, lineno, w);
            if (rc) return rc;
        }
        const int64_t ui = intern(u), vi = intern(v);
        if (ui == vi) {
            ++g->self_loops;
            continue;
        }
        g->rows.push_back(ui);
        g->cols.push_back(vi);
        g->vals.push_back(w);
        if (!directed) {
            g->rows.push_back(vi);
            g->cols.push_back(ui);
            g->vals.push_back(w);
        }
    }
    if (g->labels.empty()) return fail(DS_EPARSE, path, last > 1 ? last : 1, "no vertices found");
    g->n = (int64_t)g->labels.size();
    return DS_OK;
}

}  // namespace

extern "C" int ds_ingest_parse(const char* data, int64_t len, int32_t format, int32_t directed,
                               double default_weight, const char* name, ds_ingest** out) {
    g_err_line = 0;
    if (!out || (len > 0 && !data)) return ds_internal_set_err(DS_EINVAL, "null ingest argument");
    if (format != DS_FMT_MTX && format != DS_FMT_EDGES)
        return ds_internal_set_err(DS_EINVAL, "unknown graph format");
    const std::string path = name ? name : "-";
    ds_ingest* g = new ds_ingest();
    const int rc = format == DS_FMT_MTX
                       ? parse_mtx(data, (size_t)len, default_weight, path, g)
                       : parse_edges(data, (size_t)len, directed != 0, default_weight, path, g);
    if (rc) {
        delete g;
        *out = nullptr;
        return rc;
    }
    *out = g;
    return DS_OK;
}

extern "C" int ds_ingest_info(const ds_ingest* g, int64_t* n, int64_t* entries, int64_t* self_loops) {
    if (!g) return ds_internal_set_err(DS_EINVAL, "null ingest handle");
    if (n) *n = g->n;
    if (entries) *entries = (int64_t)g->rows.size();
    if (self_loops) *self_loops = g->self_loops;
    return DS_OK;
}

extern "C" int ds_ingest_copy(const ds_ingest* g, int64_t* rows, int64_t* cols, double* vals,
                              int64_t* labels) {
    if (!g) return ds_internal_set_err(DS_EINVAL, "null ingest handle");
    const size_t m = g->rows.size();
    if (m && rows) memcpy(rows, g->rows.data(), m * sizeof(int64_t));
    if (m && cols) memcpy(cols, g->cols.data(), m * sizeof(int64_t));
    if (m && vals) memcpy(vals, g->vals.data(), m * sizeof(double));
    if (labels && !g->labels.empty()) memcpy(labels, g->labels.data(), g->labels.size() * sizeof(int64_t));
    return DS_OK;
}

extern "C" int64_t ds_ingest_error_line(void) { return g_err_line; }

extern "C" void ds_ingest_free(ds_ingest* g) { delete g; }
