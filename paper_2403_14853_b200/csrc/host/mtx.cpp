// mtx.cpp -- on-disk formats either side of the hot path (sgnn_host.h):
// Matrix Market coordinate files (io.hpp:80-165 load_mtx, :168-185 save_mtx),
// the plain-text dense feature matrix (io.hpp:187-205) and the label / mask
// columns (io.hpp:209-262).
//
// Behaviour follows the reference loaders line for line in what they accept,
// what they reject and the message + 1-based line number they report; the
// work is split differently: the file is read once into memory, the entry
// lines are parsed by all host threads in newline-aligned chunks, and the COO
// -> CSR build is a parallel counting sort by row, a stable per-row sort by
// column and a duplicate merge -- bitwise the reference's csr_from_coo
// (sparse.hpp:26-57), see build_csr for how its std::sort order among
// duplicates is reproduced.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <new>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "../../../include/sgnn_host.h"

namespace {

constexpr int kOk = 0, kConfig = 3, kIo = 5, kParse = 6;

int n_threads(int threads) {
    if (threads > 0) return threads;
    unsigned hw = std::thread::hardware_concurrency();
    return hw ? int(hw) : 1;
}

struct Failure {
    int status = kOk;
    long line = 0;
    std::string what;
};

int report(const Failure& f, char* err, size_t err_len, long* err_line) {
    if (err && err_len) {
        const size_t n = std::min(err_len - 1, f.what.size());
        std::memcpy(err, f.what.data(), n);
        err[n] = 0;
    }
    if (err_line) *err_line = f.line;
    return f.status;
}

bool read_file(const char* path, std::string& buf) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return false;
    char tmp[1 << 16];
    size_t got;
    while ((got = std::fread(tmp, 1, sizeof tmp, f)) > 0) buf.append(tmp, got);
    const bool ok = !std::ferror(f);
    std::fclose(f);
    return ok;
}

// std::getline over an in-memory buffer: lines split at '\n' only ('\r'
// stays in the line and is whitespace to the tokenizer, as with >>).
struct LineReader {
    const char* p;
    const char* end;
    bool next(std::string_view& line) {
        if (p >= end) return false;
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', size_t(end - p)));
        const char* e = nl ? nl : end;
        line = std::string_view(p, size_t(e - p));
        p = nl ? nl + 1 : end;
        return true;
    }
};

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

// whitespace tokens (istringstream >> std::string); returns the token count,
// storing at most `cap`.
int tokenize(std::string_view s, std::string_view* out, int cap) {
    int n = 0;
    size_t i = 0;
    while (i < s.size()) {
        while (i < s.size() && is_ws(s[i])) ++i;
        if (i >= s.size()) break;
        size_t j = i;
        while (j < s.size() && !is_ws(s[j])) ++j;
        if (n < cap) out[n] = s.substr(i, j - i);
        ++n;
        i = j;
    }
    return n;
}

// std::stoll / std::stod acceptance (strtoll / strtod, whole token consumed,
// ERANGE rejected like libstdc++'s __stoa).
bool parse_index(std::string_view t, long long& out) {
    char small[64];
    std::string big;
    const char* s;
    if (t.size() < sizeof small) {
        std::memcpy(small, t.data(), t.size());
        small[t.size()] = 0;
        s = small;
    } else {
        big.assign(t);
        s = big.c_str();
    }
    char* e = nullptr;
    errno = 0;
    const long long v = std::strtoll(s, &e, 10);
    if (e == s || errno == ERANGE || size_t(e - s) != t.size()) return false;
    out = v;
    return true;
}

bool parse_value(std::string_view t, double& out) {
    char small[128];
    std::string big;
    const char* s;
    if (t.size() < sizeof small) {
        std::memcpy(small, t.data(), t.size());
        small[t.size()] = 0;
        s = small;
    } else {
        big.assign(t);
        s = big.c_str();
    }
    char* e = nullptr;
    errno = 0;
    const double v = std::strtod(s, &e);
    if (e == s || errno == ERANGE || size_t(e - s) != t.size()) return false;
    out = v;
    return true;
}

std::string lower(std::string_view s) {
    std::string r(s);
    for (char& c : r) c = char(std::tolower(static_cast<unsigned char>(c)));
    return r;
}

// newline-aligned split of [b, e) into up to t chunks
std::vector<const char*> chunk_bounds(const char* b, const char* e, int t) {
    std::vector<const char*> cut{b};
    const size_t n = size_t(e - b);
    for (int c = 1; c < t; ++c) {
        const char* p = b + n * size_t(c) / size_t(t);
        if (p < cut.back()) p = cut.back();
        const char* nl = p < e ? static_cast<const char*>(std::memchr(p, '\n', size_t(e - p))) : nullptr;
        p = nl ? nl + 1 : e;
        cut.push_back(p);
    }
    cut.push_back(e);
    return cut;
}

template <class Fn>
void run_threads(int t, Fn&& fn) {
    std::vector<std::thread> ws;
    for (int c = 1; c < t; ++c) ws.emplace_back([&, c] { fn(c); });
    fn(0);
    for (auto& w : ws) w.join();
}

// Lines of [b, e) as std::getline sees them (a final unterminated line counts).
uint64_t count_lines(const char* b, const char* e) {
    uint64_t n = 0;
    for (const char* p = b; p < e;) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', size_t(e - p)));
        ++n;
        if (!nl) break;
        p = nl + 1;
    }
    return n;
}

struct Coo {
    uint32_t row, col;
    float val;
};

struct Csr {
    uint32_t n_rows = 0, n_cols = 0;
    std::vector<uint64_t> rp;
    std::vector<uint32_t> ci;
    std::vector<float> v;
};

struct Dense {
    uint32_t rows = 0, cols = 0;
    std::vector<float> x;
};

// Per-chunk result of the parallel entry parse.
struct ChunkOut {
    std::vector<Coo> coo;
    uint64_t entries = 0;  // entry lines parsed successfully before any error
    uint64_t lines = 0;    // lines consumed up to (and including) an error line
    bool failed = false;
    std::string what;
};

// csr_from_coo (sparse.hpp:26-57) exactly as the reference orders it.
// Fast path: rows by a parallel counting sort (stable), columns by a stable
// per-row sort, duplicates summed in that order.  The reference sorts with
// std::sort, whose order among equal (row, col) keys is unspecified; since
// fp32 addition is commutative, that order only shows in the bits when a key
// occurs three or more times -- then the triples (kept in the reference's
// push order) are sorted with the very same std::sort call instead.
void merge_sorted(const Coo* sorted, uint64_t n, uint32_t n_rows, Csr& out) {
    out.rp.assign(uint64_t(n_rows) + 1, 0);
    out.ci.clear();
    out.v.clear();
    out.ci.reserve(n);
    out.v.reserve(n);
    for (uint64_t t = 0; t < n; ++t) {
        if (!out.ci.empty() && sorted[t].row == sorted[t - 1].row && sorted[t].col == sorted[t - 1].col) {
            out.v.back() += sorted[t].val;
        } else {
            out.ci.push_back(sorted[t].col);
            out.v.push_back(sorted[t].val);
        }
        out.rp[sorted[t].row + 1] = out.ci.size();
    }
    for (uint32_t i = 1; i <= n_rows; ++i) out.rp[i] = std::max(out.rp[i], out.rp[i - 1]);
}

void build_csr(std::vector<std::vector<Coo>>& parts, uint32_t n_rows, uint32_t n_cols, int t, Csr& out) {
    out.n_rows = n_rows;
    out.n_cols = n_cols;
    const int np = int(parts.size());
    std::vector<uint64_t> base(size_t(np) * (uint64_t(n_rows) + 1), 0);
    run_threads(np, [&](int c) {
        uint64_t* h = base.data() + size_t(c) * (uint64_t(n_rows) + 1);
        for (const Coo& e : parts[size_t(c)]) ++h[e.row];
    });
    // offsets: row-major over (row, part) so a row's entries keep part order
    std::vector<uint64_t> start(uint64_t(n_rows) + 1, 0);
    uint64_t run = 0;
    for (uint32_t r = 0; r < n_rows; ++r) {
        start[r] = run;
        for (int c = 0; c < np; ++c) {
            uint64_t& h = base[size_t(c) * (uint64_t(n_rows) + 1) + r];
            const uint64_t cnt = h;
            h = run;
            run += cnt;
        }
    }
    start[n_rows] = run;
    std::vector<Coo> sorted(run);
    run_threads(np, [&](int c) {
        uint64_t* h = base.data() + size_t(c) * (uint64_t(n_rows) + 1);
        for (const Coo& e : parts[size_t(c)]) sorted[h[e.row]++] = e;
    });
    std::vector<uint64_t>().swap(base);
    // per-row stable sort by column, unique counts, and the >= 3 duplicate probe
    std::vector<uint64_t> uniq(uint64_t(n_rows) + 1, 0);
    const int tt = std::max(1, std::min<int>(t, int(n_rows / 1024) + 1));
    std::vector<char> triple_dup(size_t(tt), 0);
    run_threads(tt, [&](int c) {
        const uint32_t r0 = uint32_t(uint64_t(n_rows) * c / tt), r1 = uint32_t(uint64_t(n_rows) * (c + 1) / tt);
        for (uint32_t r = r0; r < r1; ++r) {
            Coo* b = sorted.data() + start[r];
            Coo* e = sorted.data() + start[r + 1];
            std::stable_sort(b, e, [](const Coo& x, const Coo& y) { return x.col < y.col; });
            uint64_t u = 0;
            for (Coo* p = b; p < e; ++p) {
                if (p == b || p->col != p[-1].col) ++u;
                else if (p - b >= 2 && p[-2].col == p->col) triple_dup[size_t(c)] = 1;
            }
            uniq[r + 1] = u;
        }
    });
    if (std::any_of(triple_dup.begin(), triple_dup.end(), [](char f) { return f != 0; })) {
        std::vector<Coo> seq;
        seq.reserve(run);
        for (auto& p : parts) seq.insert(seq.end(), p.begin(), p.end());
        for (auto& p : parts) std::vector<Coo>().swap(p);
        std::vector<Coo>().swap(sorted);
        std::sort(seq.begin(), seq.end(),
                  [](const Coo& a, const Coo& b) { return a.row != b.row ? a.row < b.row : a.col < b.col; });
        merge_sorted(seq.data(), seq.size(), n_rows, out);
        return;
    }
    for (auto& p : parts) std::vector<Coo>().swap(p);
    out.rp.assign(uint64_t(n_rows) + 1, 0);
    for (uint32_t r = 0; r < n_rows; ++r) out.rp[r + 1] = out.rp[r] + uniq[r + 1];
    out.ci.resize(out.rp[n_rows]);
    out.v.resize(out.rp[n_rows]);
    run_threads(tt, [&](int c) {
        const uint32_t r0 = uint32_t(uint64_t(n_rows) * c / tt), r1 = uint32_t(uint64_t(n_rows) * (c + 1) / tt);
        for (uint32_t r = r0; r < r1; ++r) {
            uint64_t o = out.rp[r];
            for (uint64_t p = start[r]; p < start[r + 1]; ++p) {
                const Coo& e = sorted[p];
                if (p > start[r] && e.col == sorted[p - 1].col) {
                    out.v[o - 1] += e.val;  // T-precision accumulation (sparse.hpp:46)
                } else {
                    out.ci[o] = e.col;
                    out.v[o] = e.val;
                    ++o;
                }
            }
        }
    });
}

int load_mtx(const char* path, int threads, Csr& out, Failure& f) {
    std::string buf;
    if (!read_file(path, buf)) {
        f = {kIo, 0, std::string("cannot open '") + path + "'"};
        return kIo;
    }
    auto parse_fail = [&](const std::string& what, long line) {
        f = {kParse, line, what};
        return kParse;
    };
    LineReader rd{buf.data(), buf.data() + buf.size()};
    std::string_view line;
    long line_no = 0;
    if (!rd.next(line)) return parse_fail("missing Matrix Market banner", 1);
    ++line_no;
    std::string_view tok[8];
    const std::string low = lower(line);
    const int nb = tokenize(low, tok, 8);
    if (nb < 4 || tok[0] != "%%matrixmarket" || tok[1] != "matrix")
        return parse_fail("not a Matrix Market matrix banner", line_no);
    if (tok[2] != "coordinate")
        return parse_fail("unsupported format '" + std::string(tok[2]) + "' (only coordinate)", line_no);
    const std::string field(tok[3]);
    if (field != "real" && field != "integer" && field != "pattern")
        return parse_fail("unsupported field '" + field + "'", line_no);
    const bool pattern = field == "pattern";
    const std::string symmetry = nb > 4 ? std::string(tok[4]) : "general";
    if (symmetry != "general" && symmetry != "symmetric")
        return parse_fail("unsupported symmetry '" + symmetry + "'", line_no);
    const bool symmetric = symmetry == "symmetric";

    long long n_rows = -1, n_cols = -1, n_entries = -1;
    while (rd.next(line)) {
        ++line_no;
        if (line.empty() || line[0] == '%') continue;
        const int nt = tokenize(line, tok, 8);
        if (nt != 3 || !parse_index(tok[0], n_rows) || !parse_index(tok[1], n_cols) ||
            !parse_index(tok[2], n_entries) || n_rows < 0 || n_cols < 0 || n_entries < 0)
            return parse_fail("malformed size line '" + std::string(line) + "'", line_no);
        break;
    }
    if (n_rows < 0) return parse_fail("missing size line", line_no + 1);

    // entry lines, parsed in parallel chunks
    const char* body = rd.p;
    const char* end = buf.data() + buf.size();
    int t = n_threads(threads);
    t = int(std::max<size_t>(1, std::min<size_t>(size_t(t), size_t(end - body) / (1 << 20) + 1)));
    const auto cut = chunk_bounds(body, end, t);
    std::vector<ChunkOut> co(static_cast<size_t>(t));
    const size_t want = pattern ? 2 : 3;
    run_threads(t, [&](int c) {
        ChunkOut& o = co[size_t(c)];
        LineReader r{cut[size_t(c)], cut[size_t(c) + 1]};
        std::string_view ln, tk[4];
        while (r.next(ln)) {
            ++o.lines;
            if (ln.empty() || ln[0] == '%') continue;
            const int nt = tokenize(ln, tk, 4);
            long long rr, cc;
            double v = 1.0;
            if (size_t(nt) != want || !parse_index(tk[0], rr) || !parse_index(tk[1], cc) ||
                (!pattern && !parse_value(tk[2], v))) {
                o.failed = true;
                o.what = "malformed entry '" + std::string(ln) + "'";
                return;
            }
            if (rr < 1 || rr > n_rows || cc < 1 || cc > n_cols) {
                o.failed = true;
                o.what = "entry (" + std::to_string(rr) + ", " + std::to_string(cc) + ") out of range for " +
                         std::to_string(n_rows) + "x" + std::to_string(n_cols);
                return;
            }
            const uint32_t ri = uint32_t(rr - 1), ci = uint32_t(cc - 1);
            o.coo.push_back({ri, ci, float(v)});
            if (symmetric && ri != ci) o.coo.push_back({ci, ri, float(v)});
            ++o.entries;
        }
    });
    // stitch the chunks in file order: entries past n_entries (and anything
    // wrong with them) are never read by the reference
    uint64_t seen = 0;
    long lines_before = line_no;
    std::vector<std::vector<Coo>> parts;
    for (int c = 0; c < t && seen < uint64_t(n_entries); ++c) {
        ChunkOut& o = co[size_t(c)];
        const uint64_t take = std::min<uint64_t>(o.entries, uint64_t(n_entries) - seen);
        if (take < o.entries) {  // truncate this chunk's triples after entry `take`
            uint64_t keep = 0, got = 0;
            while (got < take) {
                const Coo& e = o.coo[keep];
                ++keep;
                const bool mirrored = symmetric && e.row != e.col;
                if (mirrored) ++keep;
                ++got;
            }
            o.coo.resize(keep);
        }
        seen += take;
        if (o.failed && seen < uint64_t(n_entries))
            return parse_fail(o.what, lines_before + long(o.lines));
        lines_before += long(o.lines);
        parts.push_back(std::move(o.coo));
    }
    if (seen < uint64_t(n_entries))
        return parse_fail("expected " + std::to_string(n_entries) + " entries, found " + std::to_string(seen),
                          line_no + long(count_lines(body, end)) + 1);
    if (uint64_t(n_rows) > 0xffffffffull || uint64_t(n_cols) > 0xffffffffull) {
        f = {kConfig, 0, "matrix dimensions exceed 32-bit indices"};
        return kConfig;
    }
    if (parts.empty()) parts.emplace_back();
    build_csr(parts, uint32_t(n_rows), uint32_t(n_cols), n_threads(threads), out);
    return kOk;
}

int load_features(const char* path, int threads, Dense& out, Failure& f) {
    std::string buf;
    if (!read_file(path, buf)) {
        f = {kIo, 0, std::string("cannot open '") + path + "'"};
        return kIo;
    }
    auto parse_fail = [&](const std::string& what, long line) {
        f = {kParse, line, what};
        return kParse;
    };
    LineReader rd{buf.data(), buf.data() + buf.size()};
    std::string_view line, tok[4];
    long line_no = 0;
    if (!rd.next(line)) return parse_fail("missing 'n k' header", 1);
    ++line_no;
    long long n, k;
    if (tokenize(line, tok, 4) != 2 || !parse_index(tok[0], n) || !parse_index(tok[1], k) || n < 0 || k < 0)
        return parse_fail("malformed header '" + std::string(line) + "' (expected 'n k')", line_no);
    out.rows = uint32_t(n);
    out.cols = uint32_t(k);
    out.x.assign(uint64_t(n) * uint64_t(k), 0.0f);
    const char* body = rd.p;
    const char* end = buf.data() + buf.size();
    int t = n_threads(threads);
    t = int(std::max<size_t>(1, std::min<size_t>(size_t(t), size_t(end - body) / (1 << 20) + 1)));
    const auto cut = chunk_bounds(body, end, t);
    struct Part {
        std::vector<float> vals;
        uint64_t rows = 0, lines = 0;
        bool failed = false;
        std::string what;
    };
    std::vector<Part> ps(static_cast<size_t>(t));
    run_threads(t, [&](int c) {
        Part& o = ps[size_t(c)];
        LineReader r{cut[size_t(c)], cut[size_t(c) + 1]};
        std::string_view ln;
        std::vector<std::string_view> tk(size_t(k) + 1);
        while (r.next(ln)) {
            ++o.lines;
            if (ln.empty()) continue;
            const int nt = tokenize(ln, tk.data(), int(k) + 1);
            if (nt != k) {
                o.failed = true;
                o.what = "row has " + std::to_string(nt) + " values, expected " + std::to_string(k);
                return;
            }
            for (long long j = 0; j < k; ++j) {
                double v;
                if (!parse_value(tk[size_t(j)], v)) {
                    o.failed = true;
                    o.what = "non-numeric value '" + std::string(tk[size_t(j)]) + "'";
                    return;
                }
                o.vals.push_back(float(v));
            }
            ++o.rows;
        }
    });
    uint64_t row = 0;
    long lines_before = line_no;
    for (int c = 0; c < t && row < uint64_t(n); ++c) {
        Part& o = ps[size_t(c)];
        const uint64_t take = std::min<uint64_t>(o.rows, uint64_t(n) - row);
        std::copy(o.vals.begin(), o.vals.begin() + ptrdiff_t(take * uint64_t(k)), out.x.begin() + ptrdiff_t(row * uint64_t(k)));
        row += take;
        if (o.failed && row < uint64_t(n)) return parse_fail(o.what, lines_before + long(o.lines));
        lines_before += long(o.lines);
    }
    if (row < uint64_t(n))
        return parse_fail("expected " + std::to_string(n) + " rows, found " + std::to_string(row),
                          line_no + long(count_lines(body, end)) + 1);
    return kOk;
}

// load_int_column (io.hpp:209-240) + the label / mask checks (:243-262)
int load_int_column(const char* path, int kind, std::vector<long long>& out, Failure& f) {
    std::string buf;
    if (!read_file(path, buf)) {
        f = {kIo, 0, std::string("cannot open '") + path + "'"};
        return kIo;
    }
    auto parse_fail = [&](const std::string& what, long line) {
        f = {kParse, line, what};
        return kParse;
    };
    LineReader rd{buf.data(), buf.data() + buf.size()};
    std::string_view line, tok[2];
    long line_no = 0;
    if (!rd.next(line)) return parse_fail("missing 'n' header", 1);
    ++line_no;
    long long n;
    if (tokenize(line, tok, 2) != 1 || !parse_index(tok[0], n) || n < 0)
        return parse_fail("malformed header '" + std::string(line) + "' (expected a count)", line_no);
    out.clear();
    while (rd.next(line)) {
        ++line_no;
        if (line.empty()) continue;
        size_t i = 0;
        while (i < line.size()) {
            while (i < line.size() && is_ws(line[i])) ++i;
            if (i >= line.size()) break;
            size_t j = i;
            while (j < line.size() && !is_ws(line[j])) ++j;
            const std::string_view t = line.substr(i, j - i);
            long long v;
            if (!parse_index(t, v)) return parse_fail("non-integer token '" + std::string(t) + "'", line_no);
            out.push_back(v);
            if (out.size() > uint64_t(n)) return parse_fail("more than " + std::to_string(n) + " values", line_no);
            i = j;
        }
    }
    if (out.size() != uint64_t(n))
        return parse_fail("expected " + std::to_string(n) + " values, found " + std::to_string(out.size()),
                          line_no + 1);
    for (size_t i = 0; i < out.size(); ++i) {
        if (kind == 0 && out[i] < 0) return parse_fail("negative label", long(i) + 2);
        if (kind == 1 && out[i] != 0 && out[i] != 1) return parse_fail("mask value must be 0 or 1", long(i) + 2);
    }
    return kOk;
}

}  // namespace

extern "C" {

int sgnn_host_mtx_load(const char* path, int threads, void** out, char* err, size_t err_len, long* err_line) {
    Failure f;
    auto* m = new Csr;
    int st;
    try {
        st = load_mtx(path, threads, *m, f);
    } catch (const std::bad_alloc&) {
        f = {kConfig, 0, "out of host memory"};
        st = kConfig;
    }
    if (st != kOk) {
        delete m;
        *out = nullptr;
        return report(f, err, err_len, err_line);
    }
    *out = m;
    return kOk;
}

void sgnn_host_csr_dims(void* h, uint32_t* n_rows, uint32_t* n_cols, uint64_t* nnz) {
    const Csr* m = static_cast<const Csr*>(h);
    *n_rows = m->n_rows;
    *n_cols = m->n_cols;
    *nnz = m->ci.size();
}

void sgnn_host_csr_export(void* h, uint64_t* rp, uint32_t* ci, float* v) {
    const Csr* m = static_cast<const Csr*>(h);
    std::memcpy(rp, m->rp.data(), m->rp.size() * sizeof(uint64_t));
    std::memcpy(ci, m->ci.data(), m->ci.size() * sizeof(uint32_t));
    std::memcpy(v, m->v.data(), m->v.size() * sizeof(float));
}

void sgnn_host_csr_free(void* h) { delete static_cast<Csr*>(h); }

int sgnn_host_mtx_save(const char* path, uint32_t n_rows, uint32_t n_cols, const uint64_t* rp,
                       const uint32_t* ci, const float* v, int threads, char* err, size_t err_len) {
    FILE* f = std::fopen(path, "wb");
    if (!f) return report({kIo, 0, std::string("cannot open '") + path + "' for writing"}, err, err_len, nullptr);
    bool ok = std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%u %u %llu\n", n_rows, n_cols,
                           static_cast<unsigned long long>(rp[n_rows])) > 0;
    // format row blocks in parallel, write them in order
    int t = std::max(1, std::min<int>(n_threads(threads), int(rp[n_rows] / 65536) + 1));
    const uint32_t block = 1u << 14;
    for (uint32_t r0 = 0; ok && r0 < n_rows; r0 += block * uint32_t(t)) {
        std::vector<std::string> out(static_cast<size_t>(t));
        run_threads(t, [&](int c) {
            const uint64_t b0 = uint64_t(r0) + uint64_t(c) * block;
            const uint64_t b1 = std::min<uint64_t>(b0 + block, n_rows);
            std::string& s = out[size_t(c)];
            char line[96];
            for (uint64_t r = b0; r < b1; ++r)
                for (uint64_t e = rp[r]; e < rp[r + 1]; ++e) {
                    const int len = std::snprintf(line, sizeof line, "%llu %u %.9g\n",
                                                  static_cast<unsigned long long>(r + 1), ci[e] + 1, double(v[e]));
                    s.append(line, size_t(len));
                }
        });
        for (const auto& s : out)
            if (!s.empty() && std::fwrite(s.data(), 1, s.size(), f) != s.size()) ok = false;
    }
    if (std::fclose(f) != 0) ok = false;
    if (!ok) return report({kIo, 0, std::string("write to '") + path + "' failed"}, err, err_len, nullptr);
    return kOk;
}

int sgnn_host_features_load(const char* path, int threads, void** out, char* err, size_t err_len,
                            long* err_line) {
    Failure f;
    auto* d = new Dense;
    int st;
    try {
        st = load_features(path, threads, *d, f);
    } catch (const std::bad_alloc&) {
        f = {kConfig, 0, "out of host memory"};
        st = kConfig;
    }
    if (st != kOk) {
        delete d;
        *out = nullptr;
        return report(f, err, err_len, err_line);
    }
    *out = d;
    return kOk;
}

void sgnn_host_dense_dims(void* h, uint32_t* rows, uint32_t* cols) {
    *rows = static_cast<Dense*>(h)->rows;
    *cols = static_cast<Dense*>(h)->cols;
}

void sgnn_host_dense_export(void* h, float* out) {
    const Dense* d = static_cast<const Dense*>(h);
    std::memcpy(out, d->x.data(), d->x.size() * sizeof(float));
}

void sgnn_host_dense_free(void* h) { delete static_cast<Dense*>(h); }

int sgnn_host_int_column_load(const char* path, int kind, uint64_t max_n, uint32_t* out, uint64_t* n,
                              char* err, size_t err_len, long* err_line) {
    Failure f;
    std::vector<long long> vals;
    if (load_int_column(path, kind, vals, f) != kOk) return report(f, err, err_len, err_line);
    *n = vals.size();
    if (out) {
        if (vals.size() > max_n) return report({kConfig, 0, "output buffer too small"}, err, err_len, err_line);
        for (size_t i = 0; i < vals.size(); ++i) out[i] = uint32_t(vals[i]);
    }
    return kOk;
}

}  // extern "C"
