// cli.cpp -- LIBSVM-style command-line front end over the C ABI (the
// drop-in use of P:52 / P:107; flags as S:464-497).  One binary, three commands:
//
//   plssvm train   [-t kernel] [-d degree] [-g gamma] [-r coef0] [-c cost] [-e eps] [-i max_iter]
//                  [--mode auto|implicit|cached] [--fp32] [-q] data_file [model_file]
//   plssvm predict [-q] test_file model_file output_file
//   plssvm scale   [-l lower] [-u upper] [-s save_ranges] [-r restore_ranges] data_file   (to stdout)
//
// (also callable as plssvm-train / plssvm-predict / plssvm-scale through symlinks).  train prints
// the paper's component breakdown (read / transform / cg / write / total) and the CG
// iteration count.  Exit codes: 0 success, 1 usage error, 2 runtime error.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "../../include/plssvm.h"

namespace {

using clk = std::chrono::steady_clock;
double secs(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

int usage(const char *msg) {
    std::fprintf(stderr,
                 "%s\nusage:\n"
                 "  plssvm train   [-t 0|1|2] [-d degree] [-g gamma] [-r coef0] [-c cost] [-e eps] [-i max_iter]\n"
                 "                 [--mode auto|implicit|cached] [--fp32] [-q] data_file [model_file]\n"
                 "  plssvm predict [-q] test_file model_file output_file\n"
                 "  plssvm scale   [-l lower] [-u upper] [-s save_file] [-r restore_file] data_file\n",
                 msg);
    return 1;
}

int runtime_error(const char *what, int status) {
    std::fprintf(stderr, "plssvm: %s failed (status %d): %s\n", what, status, plssvm_last_error());
    return 2;
}

bool need_value(int argc, char **argv, int i) { return i + 1 < argc && argv[i + 1][0] != '\0'; }

bool to_double(const char *s, double &v) {
    char *e = nullptr;
    v = std::strtod(s, &e);
    return e && *e == '\0' && e != s;
}

struct Data {
    int64_t m = 0, d = 0;
    std::vector<double> X, y;
    double labels[2] = {0.0, 0.0};
    int32_t nlabels = 0;
};

// Query, then read with row stride cap_d (>= the file's d).
int read_data(const char *path, Data &D, int64_t min_d) {
    int s = plssvm_libsvm_read(path, nullptr, nullptr, 0, 0, &D.m, &D.d, D.labels, &D.nlabels);
    if (s) return s;
    D.d = std::max<int64_t>(std::max<int64_t>(D.d, min_d), 1);
    D.X.assign(static_cast<size_t>(D.m * D.d), 0.0);
    D.y.assign(static_cast<size_t>(D.m), 0.0);
    int64_t m2, d2;
    return plssvm_libsvm_read(path, D.X.data(), D.y.data(), D.m, D.d, &m2, &d2, D.labels, &D.nlabels);
}

int cmd_train(int argc, char **argv) {
    int kernel = PLSSVM_RBF, degree = 3, mode = PLSSVM_MODE_AUTO;
    double gamma = -1.0, coef0 = 0.0, C = 1.0, eps = 1e-6;
    bool gamma_given = false;
    int64_t max_iter = 0;
    bool fp32 = false, quiet = false;
    std::vector<const char *> pos;
    for (int i = 0; i < argc; ++i) {
        const std::string a = argv[i];
        double v;
        if (a == "-q") quiet = true;
        else if (a == "--fp32") fp32 = true;
        else if (a == "--mode") {
            if (!need_value(argc, argv, i)) return usage("--mode needs a value");
            const std::string mv = argv[++i];
            if (mv == "auto") mode = PLSSVM_MODE_AUTO;
            else if (mv == "implicit") mode = PLSSVM_MODE_IMPLICIT;
            else if (mv == "cached") mode = PLSSVM_MODE_CACHED;
            else return usage("--mode must be auto, implicit or cached");
        } else if (a.size() == 2 && a[0] == '-' && std::strchr("tdgrcei", a[1])) {
            if (!need_value(argc, argv, i) || !to_double(argv[i + 1], v)) return usage(("bad value for " + a).c_str());
            ++i;
            switch (a[1]) {
                case 't':
                    if (v != 0 && v != 1 && v != 2)
                        return usage("-t must be 0 (linear), 1 (polynomial) or 2 (rbf); 3 (sigmoid) is not supported");
                    kernel = static_cast<int>(v);
                    break;
                case 'd': degree = static_cast<int>(v); break;
                case 'g': gamma = v; gamma_given = true; break;
                case 'r': coef0 = v; break;
                case 'c': C = v; break;
                case 'e': eps = v; break;
                case 'i': max_iter = static_cast<int64_t>(v); break;
            }
        } else if (!a.empty() && a[0] == '-') {
            return usage(("unknown option " + a).c_str());
        } else {
            pos.push_back(argv[i]);
        }
    }
    if (pos.empty() || pos.size() > 2) return usage("train needs data_file [model_file]");
    const std::string data = pos[0];
    const std::string model = pos.size() > 1 ? pos[1] : data + ".model";
    const auto t0 = clk::now();
    Data D;
    int s = read_data(data.c_str(), D, 1);
    if (s) return runtime_error("reading the data file", s);
    if (D.nlabels != 2) {
        std::fprintf(stderr, "plssvm: %s: training needs exactly two distinct labels (P:136-138)\n", data.c_str());
        return 2;
    }
    // first-seen label -> +1, the other -> -1
    std::vector<double> ypm(D.y.size());
    for (size_t i = 0; i < D.y.size(); ++i) ypm[i] = D.y[i] == D.labels[0] ? 1.0 : -1.0;
    // LIBSVM default 1/num_features only when -g is absent; an explicit -g <= 0 reaches the
    // library's validation ("gamma must be > 0")
    if (!gamma_given) gamma = 1.0 / static_cast<double>(D.d);
    const auto t1 = clk::now();
    plssvm_options_t o;
    plssvm_default_options(&o);
    o.mode = mode;
    o.max_iter = max_iter;
    plssvm_stats_t st;
    std::vector<double> alpha(static_cast<size_t>(D.m));
    double b = 0.0;
    if (fp32) {
        std::vector<float> Xf(D.X.begin(), D.X.end()), yf(ypm.begin(), ypm.end()), af(alpha.size());
        float bf = 0.f;
        s = plssvm_train_ex(Xf.data(), yf.data(), D.m, D.d, PLSSVM_F32, kernel, gamma, degree, coef0, C, eps, &o,
                            af.data(), &bf, &st);
        for (size_t i = 0; i < af.size(); ++i) alpha[i] = af[i];
        b = bf;
    } else {
        s = plssvm_train_ex(D.X.data(), ypm.data(), D.m, D.d, PLSSVM_F64, kernel, gamma, degree, coef0, C, eps, &o,
                            alpha.data(), &b, &st);
    }
    if (s != PLSSVM_OK && s != PLSSVM_W_NOT_CONVERGED) return runtime_error("training", s);
    const int train_status = s;
    const auto t2 = clk::now();
    s = plssvm_model_write(model.c_str(), kernel, gamma, degree, coef0, D.X.data(), alpha.data(), b, D.m, D.d,
                           ypm.data(), D.labels);
    if (s) return runtime_error("writing the model", s);
    const auto t3 = clk::now();
    if (!quiet) {
        std::printf("read %d x %d points/features from '%s', labels %g -> +1, %g -> -1\n", static_cast<int>(D.m),
                    static_cast<int>(D.d), data.c_str(), D.labels[0], D.labels[1]);
        std::printf("kernel %d gamma %.6g degree %d coef0 %g C %g eps %g mode %s%s\n", kernel, gamma, degree, coef0, C,
                    eps, st.mode_used == PLSSVM_MODE_CACHED ? "cached" : "implicit", fp32 ? " fp32" : "");
        std::printf("CG iterations %lld (residual %.3e)%s\n", static_cast<long long>(st.iterations), st.rel_residual,
                    train_status == PLSSVM_W_NOT_CONVERGED ? " NOT CONVERGED" : "");
        std::printf("read %.6f s | transform %.6f s | precompute %.6f s | cg %.6f s | write %.6f s | total %.6f s\n",
                    secs(t0, t1), st.t_h2d + st.t_transform + st.t_q, st.t_precompute, st.t_cg, secs(t2, t3),
                    secs(t0, t3));
        std::printf("model written to '%s'\n", model.c_str());
    }
    return 0;
}

int cmd_predict(int argc, char **argv) {
    bool quiet = false;
    std::vector<const char *> pos;
    for (int i = 0; i < argc; ++i) {
        if (!std::strcmp(argv[i], "-q")) quiet = true;
        else if (argv[i][0] == '-' && argv[i][1] != '\0') return usage((std::string("unknown option ") + argv[i]).c_str());
        else pos.push_back(argv[i]);
    }
    if (pos.size() != 3) return usage("predict needs test_file model_file output_file");
    int32_t kernel, degree;
    double gamma, coef0, b, labels[2];
    int64_t m, dm;
    int s = plssvm_model_read(pos[1], &kernel, &gamma, &degree, &coef0, nullptr, nullptr, &b, 0, 0, &m, &dm, labels);
    if (s) return runtime_error("reading the model", s);
    Data T;
    s = plssvm_libsvm_read(pos[0], nullptr, nullptr, 0, 0, &T.m, &T.d, T.labels, &T.nlabels);
    if (s) return runtime_error("reading the test file", s);
    const int64_t D = std::max<int64_t>(std::max(dm, T.d), 1);  // common zero-padded width
    std::vector<double> SV(static_cast<size_t>(m * D)), alpha(static_cast<size_t>(m));
    s = plssvm_model_read(pos[1], &kernel, &gamma, &degree, &coef0, SV.data(), alpha.data(), &b, m, D, &m, &dm, labels);
    if (s) return runtime_error("reading the model", s);
    s = read_data(pos[0], T, D);
    if (s) return runtime_error("reading the test file", s);
    std::vector<double> f(static_cast<size_t>(T.m));
    std::vector<int32_t> lab(static_cast<size_t>(T.m));
    s = plssvm_predict(SV.data(), alpha.data(), b, m, D, kernel, gamma, degree, coef0, T.X.data(), T.m, f.data(),
                       lab.data());
    if (s) return runtime_error("prediction", s);
    std::FILE *out = std::fopen(pos[2], "wb");
    if (!out) {
        std::fprintf(stderr, "plssvm: cannot open '%s' for writing\n", pos[2]);
        return 2;
    }
    int64_t correct = 0;
    for (int64_t i = 0; i < T.m; ++i) {
        const double l = lab[i] > 0 ? labels[0] : labels[1];
        std::fprintf(out, "%.17g\n", l);
        correct += (l == T.y[i]);
    }
    if (std::fclose(out) != 0) {
        std::fprintf(stderr, "plssvm: cannot write '%s'\n", pos[2]);
        return 2;
    }
    if (!quiet)
        std::printf("Accuracy = %.4g%% (%lld/%lld)\n", 100.0 * static_cast<double>(correct) / static_cast<double>(T.m),
                    static_cast<long long>(correct), static_cast<long long>(T.m));
    return 0;
}

// svm-scale range file: "x", "<lower> <upper>", then "<index> <min> <max>" per feature.
int cmd_scale(int argc, char **argv) {
    double lo = -1.0, hi = 1.0;
    const char *save = nullptr, *restore = nullptr;
    std::vector<const char *> pos;
    for (int i = 0; i < argc; ++i) {
        const std::string a = argv[i];
        if ((a == "-l" || a == "-u") && need_value(argc, argv, i)) {
            double v;
            if (!to_double(argv[++i], v)) return usage(("bad value for " + a).c_str());
            (a == "-l" ? lo : hi) = v;
        } else if (a == "-s" && need_value(argc, argv, i)) {
            save = argv[++i];
        } else if (a == "-r" && need_value(argc, argv, i)) {
            restore = argv[++i];
        } else if (!a.empty() && a[0] == '-') {
            return usage(("bad option " + a).c_str());
        } else {
            pos.push_back(argv[i]);
        }
    }
    if (pos.size() != 1) return usage("scale needs one data_file");
    if (save && restore) return usage("-s and -r are exclusive");
    Data D;
    std::vector<double> fmin, fmax;
    if (restore) {
        std::ifstream in(restore);
        std::string x;
        if (!(in >> x) || x != "x" || !(in >> lo >> hi)) {
            std::fprintf(stderr, "plssvm: '%s' is not a range file\n", restore);
            return 2;
        }
        int64_t k;
        double a, b;
        while (in >> k >> a >> b) {
            if (k < 1) {
                std::fprintf(stderr, "plssvm: '%s': bad feature index %lld\n", restore, static_cast<long long>(k));
                return 2;
            }
            if (static_cast<int64_t>(fmin.size()) < k) {
                fmin.resize(static_cast<size_t>(k), 0.0);
                fmax.resize(static_cast<size_t>(k), 0.0);
            }
            fmin[k - 1] = a;
            fmax[k - 1] = b;
        }
    }
    int s = read_data(pos[0], D, static_cast<int64_t>(fmin.size()));
    if (s) return runtime_error("reading the data file", s);
    if (!restore) {
        fmin.assign(static_cast<size_t>(D.d), 0.0);
        fmax.assign(static_cast<size_t>(D.d), 0.0);
        s = plssvm_scale_fit(D.X.data(), D.m, D.d, fmin.data(), fmax.data());
        if (s) return runtime_error("scale_fit", s);
    } else if (static_cast<int64_t>(fmin.size()) < D.d) {  // features absent from the range file: constant -> lo
        fmin.resize(static_cast<size_t>(D.d), 0.0);
        fmax.resize(static_cast<size_t>(D.d), 0.0);
    }
    s = plssvm_scale_apply(D.X.data(), D.m, D.d, fmin.data(), fmax.data(), lo, hi);
    if (s) return runtime_error("scale_apply", s);
    if (save) {
        std::FILE *f = std::fopen(save, "wb");
        if (!f) {
            std::fprintf(stderr, "plssvm: cannot open '%s' for writing\n", save);
            return 2;
        }
        std::fprintf(f, "x\n%.17g %.17g\n", lo, hi);
        for (int64_t k = 0; k < D.d; ++k) std::fprintf(f, "%lld %.17g %.17g\n", static_cast<long long>(k + 1), fmin[k], fmax[k]);
        std::fclose(f);
    }
    s = plssvm_libsvm_write("/dev/stdout", D.X.data(), D.y.data(), D.m, D.d);
    if (s) return runtime_error("writing the scaled data", s);
    return 0;
}

}  // namespace

int main(int argc, char **argv) {
    std::string prog = argv[0];
    const size_t sl = prog.rfind('/');
    if (sl != std::string::npos) prog = prog.substr(sl + 1);
    std::string cmd;
    int first = 1;
    if (prog == "plssvm-train") cmd = "train";
    else if (prog == "plssvm-predict") cmd = "predict";
    else if (prog == "plssvm-scale") cmd = "scale";
    else if (argc > 1) {
        cmd = argv[1];
        first = 2;
    }
    if (cmd == "train") return cmd_train(argc - first, argv + first);
    if (cmd == "predict") return cmd_predict(argc - first, argv + first);
    if (cmd == "scale") return cmd_scale(argc - first, argv + first);
    return usage("unknown command (train, predict, scale)");
}
