// io.cpp -- the steps either side of the hot path: LIBSVM data files,
// LIBSVM c_svc model files and svm-scale feature scaling, so the library is the "drop-in
// replacement for LIBSVM" of P:52 / P:107 and covers the read / write components of the
// paper's runtime breakdown (Fig. 2).  Host-only native C++ (no GPU needed).
//
// Data format: one point per line "<label> <index>:<value> ...", 1-based strictly
// ascending indices, blank and '#' lines skipped, LF or CRLF; absent features are 0 -- the data
// are treated as dense ("treated as if they would represent dense data").  The parse is
// multi-threaded: the file is read once, cut into newline-aligned chunks, each chunk parsed into
// (label, index, value) runs by its own thread, then the dense matrix is filled in parallel.
// Numbers go through std::from_chars (correctly rounded), so a file written with %.17g
// round-trips bit-exactly.
//
// Model format (LIBSVM c_svc): header svm_type / kernel_type / degree / gamma / coef0
// (as the kernel needs them) / nr_class 2 / total_sv m / rho -b / label l+ l- / nr_sv n+ n- / SV,
// then one line per training point "<alpha_i> <k>:<x_ik> ..." (zero features omitted) -- every
// LS-SVM point is a support vector; the y = +1 points first (LIBSVM groups SVs by class), each
// group in input order.  LIBSVM's decision value sum coef_i k(x_i, z) - rho is then our
// f(z) = sum alpha_i k(x_i, z) + b (Eq. 10 with labels absorbed, R-2).
//
// Scaling (svm-scale, "scaled to values between [-1, 1]"): x -> lo + (hi - lo)
// (x - min_k) / (max_k - min_k) per feature k over all points (zeros included), constant features
// -> lo, no clamping when applied to other data.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "../../include/plssvm.h"
#include "common.cuh"
#include "io.h"

namespace plssvm {
namespace io {

namespace {

[[noreturn]] void io_error(const std::string &msg) { throw Error(PLSSVM_E_IO, msg); }

std::string read_file(const char *path) {
    if (!path) throw Error(PLSSVM_E_INVALID_ARG, "NULL path");
    std::ifstream f(path, std::ios::binary);
    if (!f) io_error(std::string("cannot open '") + path + "'");
    std::string buf;
    f.seekg(0, std::ios::end);
    const std::streamoff n = f.tellg();
    if (n < 0) io_error(std::string("cannot read '") + path + "'");
    buf.resize(static_cast<size_t>(n));
    f.seekg(0, std::ios::beg);
    if (n > 0 && !f.read(&buf[0], n)) io_error(std::string("cannot read '") + path + "'");
    return buf;
}

void write_file(const char *path, const std::string &text) {
    if (!path) throw Error(PLSSVM_E_INVALID_ARG, "NULL path");
    std::FILE *f = std::fopen(path, "wb");
    if (!f) io_error(std::string("cannot open '") + path + "' for writing");
    const bool ok = std::fwrite(text.data(), 1, text.size(), f) == text.size();
    if (std::fclose(f) != 0 || !ok) io_error(std::string("cannot write '") + path + "'");
}

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// A real number token [p, e): optional leading '+' (from_chars rejects it), the rest must be a
// complete floating-point literal, finite.
bool parse_real(const char *p, const char *e, double &v) {
    if (p < e && *p == '+') ++p;
    if (p >= e) return false;
    auto r = std::from_chars(p, e, v);
    return r.ec == std::errc() && r.ptr == e && std::isfinite(v);
}

bool parse_index(const char *p, const char *e, int64_t &v) {
    if (p < e && *p == '+') ++p;
    if (p >= e) return false;
    auto r = std::from_chars(p, e, v);
    return r.ec == std::errc() && r.ptr == e;
}

// %.17g with "-0" normalised to "0"
std::string num(double v) {
    if (v == 0.0) v = 0.0;
    char b[40];
    std::snprintf(b, sizeof(b), "%.17g", v);
    return b;
}

struct Chunk {
    const char *b = nullptr, *e = nullptr;
    int64_t first_line = 1;                 // 1-based line number of the chunk's first line
    std::vector<double> label;              // per point
    std::vector<int64_t> start;             // per point: offset into idx/val (+ final sentinel)
    std::vector<int64_t> idx;
    std::vector<double> val;
    int64_t maxidx = 0;
    std::vector<double> distinct;           // first-seen order, at most 3 kept
    std::string err;
};

// Parse the lines of one chunk.  Line syntax errors are recorded with their global line number.
void parse_chunk(Chunk &c) {
    const char *p = c.b;
    int64_t line = c.first_line;
    while (p < c.e && c.err.empty()) {
        const char *le = static_cast<const char *>(std::memchr(p, '\n', static_cast<size_t>(c.e - p)));
        if (!le) le = c.e;
        const char *q = p;
        while (q < le && is_space(*q)) ++q;
        if (q < le && *q != '#') {
            // label
            const char *t = q;
            while (t < le && !is_space(*t)) ++t;
            double lab;
            if (!parse_real(q, t, lab)) {
                c.err = "line " + std::to_string(line) + ": invalid label '" + std::string(q, t) + "'";
                break;
            }
            if (std::find(c.distinct.begin(), c.distinct.end(), lab) == c.distinct.end() && c.distinct.size() < 3)
                c.distinct.push_back(lab);
            c.start.push_back(static_cast<int64_t>(c.idx.size()));
            c.label.push_back(lab);
            int64_t prev = 0;
            q = t;
            while (true) {
                while (q < le && is_space(*q)) ++q;
                if (q >= le) break;
                t = q;
                while (t < le && !is_space(*t)) ++t;
                const char *colon = static_cast<const char *>(std::memchr(q, ':', static_cast<size_t>(t - q)));
                int64_t k;
                double v;
                if (!colon || !parse_index(q, colon, k)) {
                    c.err = "line " + std::to_string(line) + ": invalid feature '" + std::string(q, t) +
                            "' (expected <index>:<value>)";
                    break;
                }
                if (k < 1) {
                    c.err = "line " + std::to_string(line) + ": feature index " + std::to_string(k) + " < 1";
                    break;
                }
                if (k <= prev) {
                    c.err = "line " + std::to_string(line) + ": indices must be ascending (" + std::to_string(k) +
                            " after " + std::to_string(prev) + ")";
                    break;
                }
                if (!parse_real(colon + 1, t, v)) {
                    c.err = "line " + std::to_string(line) + ": invalid value '" + std::string(colon + 1, t) + "'";
                    break;
                }
                prev = k;
                c.idx.push_back(k);
                c.val.push_back(v);
                q = t;
            }
            c.maxidx = std::max(c.maxidx, prev);
        }
        p = le + 1;
        ++line;
    }
    c.start.push_back(static_cast<int64_t>(c.idx.size()));
}

int num_workers(size_t bytes) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t by_size = bytes / (1u << 20) + 1;  // >= 1 MiB per thread
    return static_cast<int>(std::min<size_t>({hw, by_size, 64}));
}

template <typename F>
void parallel_for(int n, F f) {
    if (n <= 1) {
        for (int i = 0; i < n; ++i) f(i);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(n);
    for (int i = 0; i < n; ++i) th.emplace_back(f, i);
    for (auto &t : th) t.join();
}

struct Parsed {
    std::string text;
    std::vector<Chunk> chunks;
    int64_t m = 0, d = 0;
    std::vector<double> labels;  // distinct, first-seen order
};

void parse_libsvm_file(const char *path, Parsed &P) {
    P.text = read_file(path);
    const char *b = P.text.data(), *e = b + P.text.size();
    const int nw = num_workers(P.text.size());
    std::vector<const char *> cut(nw + 1, e);
    cut[0] = b;
    for (int i = 1; i < nw; ++i) {
        const char *c = b + P.text.size() * i / nw;
        c = std::max(c, cut[i - 1]);
        const char *nl = static_cast<const char *>(std::memchr(c, '\n', static_cast<size_t>(e - c)));
        cut[i] = nl ? nl + 1 : e;
    }
    P.chunks.assign(nw, Chunk());
    std::vector<int64_t> lines(nw, 0);
    parallel_for(nw, [&](int i) { lines[i] = std::count(cut[i], cut[i + 1], '\n'); });
    int64_t first = 1;
    for (int i = 0; i < nw; ++i) {
        P.chunks[i].b = cut[i];
        P.chunks[i].e = cut[i + 1];
        P.chunks[i].first_line = first;
        first += lines[i];
    }
    parallel_for(nw, [&](int i) { parse_chunk(P.chunks[i]); });
    for (auto &c : P.chunks) {
        if (!c.err.empty()) io_error(std::string(path) + ": " + c.err);
        P.m += static_cast<int64_t>(c.label.size());
        P.d = std::max(P.d, c.maxidx);
        for (double l : c.distinct)
            if (std::find(P.labels.begin(), P.labels.end(), l) == P.labels.end()) P.labels.push_back(l);
    }
    if (P.m == 0) io_error(std::string(path) + ": no data points");
    if (P.labels.size() > 2) {
        // the first line that introduces a third label, for the message
        std::vector<double> seen;
        for (auto &c : P.chunks)
            for (double l : c.label)
                if (std::find(seen.begin(), seen.end(), l) == seen.end()) {
                    seen.push_back(l);
                    if (seen.size() == 3)
                        throw Error(PLSSVM_E_LABELS, std::string(path) + ": more than two distinct labels (" + num(seen[0]) +
                                                         ", " + num(seen[1]) + ", " + num(seen[2]) +
                                                         "): PLSSVM is a binary classifier (P:136-138)");
                }
    }
}

void fill_dense(const Parsed &P, double *X, double *y, int64_t cap_d) {
    std::vector<int64_t> row0(P.chunks.size(), 0);
    for (size_t i = 1; i < P.chunks.size(); ++i) row0[i] = row0[i - 1] + static_cast<int64_t>(P.chunks[i - 1].label.size());
    parallel_for(static_cast<int>(P.chunks.size()), [&](int ci) {
        const Chunk &c = P.chunks[ci];
        for (size_t r = 0; r < c.label.size(); ++r) {
            const int64_t i = row0[ci] + static_cast<int64_t>(r);
            double *row = X + i * cap_d;
            std::fill(row, row + cap_d, 0.0);
            for (int64_t k = c.start[r]; k < c.start[r + 1]; ++k) row[c.idx[k] - 1] = c.val[k];
            y[i] = c.label[r];
        }
    });
}

void append_sparse_row(std::string &out, const double *row, int64_t d) {
    for (int64_t k = 0; k < d; ++k)
        if (row[k] != 0.0) {
            out += ' ';
            out += std::to_string(k + 1);
            out += ':';
            out += num(row[k]);
        }
}

const char *kernel_name(int kernel) {
    switch (kernel) {
        case PLSSVM_LINEAR: return "linear";
        case PLSSVM_POLYNOMIAL: return "polynomial";
        case PLSSVM_RBF: return "rbf";
        default: return nullptr;
    }
}

}  // namespace

void libsvm_read(const char *path, double *X, double *y, int64_t cap_m, int64_t cap_d, int64_t *m, int64_t *d,
                 double *labels, int32_t *nlabels) {
    Parsed P;
    parse_libsvm_file(path, P);
    if (m) *m = P.m;
    if (d) *d = P.d;
    if (labels)
        for (size_t i = 0; i < P.labels.size(); ++i) labels[i] = P.labels[i];
    if (nlabels) *nlabels = static_cast<int32_t>(P.labels.size());
    if (!X || !y) return;  // query mode
    if (cap_m < P.m || cap_d < std::max<int64_t>(P.d, 1))
        throw Error(PLSSVM_E_INVALID_ARG, "libsvm_read: buffers too small (" + std::to_string(cap_m) + " x " +
                                              std::to_string(cap_d) + " for " + std::to_string(P.m) + " x " +
                                              std::to_string(P.d) + ")");
    fill_dense(P, X, y, cap_d);
}

void libsvm_write(const char *path, const double *X, const double *y, int64_t m, int64_t d) {
    std::string out;
    out.reserve(static_cast<size_t>(m) * static_cast<size_t>(std::min<int64_t>(d, 64)) * 12 + 64);
    for (int64_t i = 0; i < m; ++i) {
        out += num(y[i]);
        append_sparse_row(out, X + i * d, d);
        out += '\n';
    }
    write_file(path, out);
}

void model_write(const char *path, int kernel, double gamma, int degree, double coef0, const double *X,
                 const double *alpha, double b, int64_t m, int64_t d, const double *y, const double *labels) {
    const char *kn = kernel_name(kernel);
    if (!kn) throw Error(PLSSVM_E_INVALID_ARG, "model_write: kernel must be 0, 1 or 2");
    int64_t npos = 0;
    for (int64_t i = 0; i < m; ++i) {
        if (y[i] != 1.0 && y[i] != -1.0) throw Error(PLSSVM_E_LABELS, "model_write: y must be +1 / -1");
        npos += y[i] == 1.0;
    }
    std::string out = "svm_type c_svc\nkernel_type ";
    out += kn;
    out += '\n';
    if (kernel == PLSSVM_POLYNOMIAL) out += "degree " + std::to_string(degree) + "\n";
    if (kernel != PLSSVM_LINEAR) out += "gamma " + num(gamma) + "\n";
    if (kernel == PLSSVM_POLYNOMIAL) out += "coef0 " + num(coef0) + "\n";
    out += "nr_class 2\ntotal_sv " + std::to_string(m) + "\n";
    out += "rho " + num(-b) + "\n";
    out += "label " + num(labels[0]) + " " + num(labels[1]) + "\n";
    out += "nr_sv " + std::to_string(npos) + " " + std::to_string(m - npos) + "\nSV\n";
    for (int pass = 0; pass < 2; ++pass)  // y = +1 points first, then y = -1 (LIBSVM's class grouping)
        for (int64_t i = 0; i < m; ++i)
            if ((y[i] == 1.0) == (pass == 0)) {
                out += num(alpha[i]);
                append_sparse_row(out, X + i * d, d);
                out += '\n';
            }
    write_file(path, out);
}

void model_read(const char *path, int32_t *kernel, double *gamma, int32_t *degree, double *coef0, double *X,
                double *alpha, double *b, int64_t cap_m, int64_t cap_d, int64_t *m, int64_t *d, double *labels) {
    const std::string text = read_file(path);
    std::istringstream in(text);
    std::string line, key;
    int kern = -1, deg = 3, nclass = -1;
    double g = 0.0, r = 0.0, rho = 0.0, lab[2] = {0.0, 0.0};
    bool have_rho = false, have_label = false, have_sv = false, have_gamma = false;
    int64_t total = -1, lineno = 0;
    auto bad = [&](const std::string &what) { io_error(std::string(path) + ": line " + std::to_string(lineno) + ": " + what); };
    auto real = [&](std::istringstream &ls, double &v) {
        std::string tok;
        if (!(ls >> tok) || !parse_real(tok.data(), tok.data() + tok.size(), v)) bad("invalid number in '" + line + "'");
    };
    while (std::getline(in, line)) {
        ++lineno;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        std::istringstream ls(line);
        if (!(ls >> key)) continue;
        if (key == "SV") {
            have_sv = true;
            break;
        } else if (key == "svm_type") {
            std::string t;
            ls >> t;
            if (t != "c_svc") bad("svm_type '" + t + "' is not supported (c_svc only)");
        } else if (key == "kernel_type") {
            std::string t;
            ls >> t;
            if (t == "linear") kern = PLSSVM_LINEAR;
            else if (t == "polynomial") kern = PLSSVM_POLYNOMIAL;
            else if (t == "rbf") kern = PLSSVM_RBF;
            else bad("unknown kernel_type '" + t + "' (linear, polynomial, rbf)");
        } else if (key == "degree") {
            double v;
            real(ls, v);
            deg = static_cast<int>(v);
            if (v != deg) bad("degree must be an integer");
        } else if (key == "gamma") {
            real(ls, g);
            have_gamma = true;
        } else if (key == "coef0") {
            real(ls, r);
        } else if (key == "nr_class") {
            double v;
            real(ls, v);
            nclass = static_cast<int>(v);
            if (nclass != 2) bad("nr_class " + std::to_string(nclass) + " is not supported (binary classification)");
        } else if (key == "total_sv") {
            double v;
            real(ls, v);
            total = static_cast<int64_t>(v);
        } else if (key == "rho") {
            real(ls, rho);
            have_rho = true;
        } else if (key == "label") {
            real(ls, lab[0]);
            real(ls, lab[1]);
            have_label = true;
        } else if (key == "nr_sv" || key == "probA" || key == "probB") {
            // informational (nr_sv: class grouping of the SV lines)
        } else {
            double v;
            if (parse_real(key.data(), key.data() + key.size(), v)) bad("missing 'SV' line before the support vectors");
            bad("unknown header field '" + key + "'");
        }
    }
    if (!have_sv) io_error(std::string(path) + ": missing 'SV' line");
    if (kern < 0) io_error(std::string(path) + ": missing field 'kernel_type'");
    if (nclass < 0) io_error(std::string(path) + ": missing field 'nr_class'");
    if (!have_rho) io_error(std::string(path) + ": missing field 'rho'");
    if (!have_label) io_error(std::string(path) + ": missing field 'label'");
    if (total < 0) io_error(std::string(path) + ": missing field 'total_sv'");
    if (kern != PLSSVM_LINEAR && !have_gamma) io_error(std::string(path) + ": missing field 'gamma'");
    // SV section: "<alpha> idx:val ..." -- same token rules as the data format
    const size_t off = static_cast<size_t>(in.tellg() < 0 ? text.size() : static_cast<size_t>(in.tellg()));
    Chunk c;
    c.b = text.data() + std::min(off, text.size());
    c.e = text.data() + text.size();
    c.first_line = lineno + 1;
    parse_chunk(c);
    if (!c.err.empty()) io_error(std::string(path) + ": " + c.err);
    const int64_t nsv = static_cast<int64_t>(c.label.size());
    if (nsv != total)
        io_error(std::string(path) + ": total_sv " + std::to_string(total) + " but " + std::to_string(nsv) + " SV lines");
    if (kernel) *kernel = kern;
    if (gamma) *gamma = g;
    if (degree) *degree = deg;
    if (coef0) *coef0 = r;
    if (b) *b = rho == 0.0 ? 0.0 : -rho;
    if (labels) {
        labels[0] = lab[0];
        labels[1] = lab[1];
    }
    if (m) *m = nsv;
    if (d) *d = c.maxidx;
    if (!X || !alpha) return;  // query mode
    if (cap_m < nsv || cap_d < std::max<int64_t>(c.maxidx, 1))
        throw Error(PLSSVM_E_INVALID_ARG, "model_read: buffers too small");
    for (int64_t i = 0; i < nsv; ++i) {
        double *row = X + i * cap_d;
        std::fill(row, row + cap_d, 0.0);
        for (int64_t k = c.start[i]; k < c.start[i + 1]; ++k) row[c.idx[k] - 1] = c.val[k];
        alpha[i] = c.label[i];
    }
}

void scale_fit(const double *X, int64_t m, int64_t d, double *fmin, double *fmax) {
    for (int64_t k = 0; k < d; ++k) {
        fmin[k] = X[k];
        fmax[k] = X[k];
    }
    for (int64_t i = 1; i < m; ++i)
        for (int64_t k = 0; k < d; ++k) {
            const double v = X[i * d + k];
            fmin[k] = std::min(fmin[k], v);
            fmax[k] = std::max(fmax[k], v);
        }
}

void scale_apply(double *X, int64_t m, int64_t d, const double *fmin, const double *fmax, double lo, double hi) {
    for (int64_t i = 0; i < m; ++i)
        for (int64_t k = 0; k < d; ++k) {
            double &v = X[i * d + k];
            v = (fmax[k] == fmin[k]) ? lo : lo + (hi - lo) * (v - fmin[k]) / (fmax[k] - fmin[k]);
        }
}

}  // namespace io
}  // namespace plssvm
