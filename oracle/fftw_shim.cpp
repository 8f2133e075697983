// Test infrastructure (oracle) -- NOT part of the product path.
//
// fp64 restatement of the two FFTW3 entry points the reference uses
// (proj/core/src/propagation.cpp:27-30 plan, :38-39 execute).  See fftw3.h for
// the contract.  Algorithm: mixed-radix Stockham autosort (radices 4,2,3,5,7
// and any prime <= 64 through a generic small DFT), Bluestein chirp-z for
// lengths with a prime factor > 64.  Single-threaded like the reference's
// FFTW usage (no fftw_init_threads anywhere in the reference).
#include "fftw3.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <memory>
#include <vector>

namespace {

using cd = std::complex<double>;
constexpr double kTwoPi = 6.283185307179586476925286766559;

struct Fft1d {
    int n = 0;
    int sign = -1;
    std::vector<int> radices;
    std::vector<cd> w;  // w[k] = exp(sign * 2 pi i k / n)
    std::vector<std::vector<cd>> small;  // per distinct radix: exp(sign 2 pi i q / r)
    // Bluestein
    bool blue = false;
    int m = 0;
    std::vector<cd> chirp;   // c_k = exp(sign * pi i k^2 / n)
    std::vector<cd> bspec;   // FFT_m of the conjugate chirp kernel
    std::unique_ptr<Fft1d> fwd_m, inv_m;

    void init(int n_, int sign_) {
        n = n_;
        sign = sign_;
        int rest = n;
        radices.clear();
        while (rest % 4 == 0) { radices.push_back(4); rest /= 4; }
        while (rest % 2 == 0) { radices.push_back(2); rest /= 2; }
        for (int p = 3; p <= 64 && rest > 1; p += 2)
            while (rest % p == 0) { radices.push_back(p); rest /= p; }
        if (rest > 1) {
            blue = true;
            m = 1;
            while (m < 2 * n - 1) m <<= 1;
            chirp.resize(n);
            for (int k = 0; k < n; ++k) {
                const uint64_t q = (static_cast<uint64_t>(k) * k) % (2ULL * n);
                const double a = sign * kTwoPi * 0.5 * static_cast<double>(q) / n;
                chirp[k] = cd(std::cos(a), std::sin(a));
            }
            fwd_m = std::make_unique<Fft1d>();
            inv_m = std::make_unique<Fft1d>();
            fwd_m->init(m, -1);
            inv_m->init(m, +1);
            std::vector<cd> b(m, cd(0.0, 0.0)), scratch(m);
            b[0] = std::conj(chirp[0]);
            for (int k = 1; k < n; ++k) b[k] = b[m - k] = std::conj(chirp[k]);
            fwd_m->run(b.data(), scratch.data());
            bspec = b;
            return;
        }
        w.resize(n);
        for (int k = 0; k < n; ++k) {
            const double a = sign * kTwoPi * static_cast<double>(k) / n;
            w[k] = cd(std::cos(a), std::sin(a));
        }
        small.assign(65, {});
        for (int r : radices) {
            if (!small[r].empty()) continue;
            small[r].resize(r);
            for (int q = 0; q < r; ++q) {
                const double a = sign * kTwoPi * static_cast<double>(q) / r;
                small[r][q] = cd(std::cos(a), std::sin(a));
            }
        }
    }

    // In-place transform of data[0..n); scratch must hold max(n, 2m) values.
    void run(cd* data, cd* scratch) const {
        if (n == 1) return;
        if (blue) {
            std::vector<cd> a(m, cd(0.0, 0.0)), s2(m);
            for (int k = 0; k < n; ++k) a[k] = data[k] * chirp[k];
            fwd_m->run(a.data(), s2.data());
            for (int k = 0; k < m; ++k) a[k] *= bspec[k];
            inv_m->run(a.data(), s2.data());
            const double inv = 1.0 / m;
            for (int k = 0; k < n; ++k) data[k] = a[k] * inv * chirp[k];
            return;
        }
        cd* in = data;
        cd* out = scratch;
        int ns = 1;
        cd v[64], y[64];
        for (int r : radices) {
            const int stride = n / r;
            const int span = n / (ns * r);
            const std::vector<cd>& tw = small[r];
            for (int j = 0; j < stride; ++j) {
                const int k = j % ns;
                for (int q = 0; q < r; ++q) v[q] = in[j + q * stride];
                if (ns > 1)
                    for (int q = 1; q < r; ++q)
                        v[q] *= w[(static_cast<int64_t>(q) * k * span) % n];
                if (r == 2) {
                    y[0] = v[0] + v[1];
                    y[1] = v[0] - v[1];
                } else if (r == 4) {
                    const cd a0 = v[0] + v[2], a1 = v[0] - v[2];
                    const cd b0 = v[1] + v[3], b1 = v[1] - v[3];
                    const cd jb1 = cd(-sign * b1.imag(), sign * b1.real());  // sign*i*b1
                    y[0] = a0 + b0;
                    y[2] = a0 - b0;
                    y[1] = a1 + jb1;
                    y[3] = a1 - jb1;
                } else {
                    for (int o = 0; o < r; ++o) {
                        cd s(0.0, 0.0);
                        for (int q = 0; q < r; ++q) s += v[q] * tw[(q * o) % r];
                        y[o] = s;
                    }
                }
                const int base = (j / ns) * ns * r + k;
                for (int q = 0; q < r; ++q) out[base + q * ns] = y[q];
            }
            ns *= r;
            std::swap(in, out);
        }
        if (in != data) std::memcpy(data, in, sizeof(cd) * n);
    }
};

}  // namespace

struct fftw_plan_s {
    int n0 = 0, n1 = 0;
    Fft1d rows, cols;
    fftw_complex* in = nullptr;
    fftw_complex* out = nullptr;
};

extern "C" {

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned /*flags*/) {
    if (n0 <= 0 || n1 <= 0 || (sign != FFTW_FORWARD && sign != FFTW_BACKWARD)) return nullptr;
    auto* p = new fftw_plan_s;
    p->n0 = n0;
    p->n1 = n1;
    p->rows.init(n1, sign);
    p->cols.init(n0, sign);
    p->in = in;
    p->out = out;
    return p;
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    const int n0 = p->n0, n1 = p->n1;
    cd* data = reinterpret_cast<cd*>(out);
    if (in != out) std::memcpy(out, in, sizeof(cd) * static_cast<size_t>(n0) * n1);
    const int big = std::max(n0, n1);
    std::vector<cd> scratch(static_cast<size_t>(big));
    for (int y = 0; y < n0; ++y) p->rows.run(data + static_cast<size_t>(y) * n1, scratch.data());
    constexpr int kBlock = 16;
    std::vector<cd> col(static_cast<size_t>(kBlock) * n0);
    for (int x0 = 0; x0 < n1; x0 += kBlock) {
        const int bw = std::min(kBlock, n1 - x0);
        for (int y = 0; y < n0; ++y)
            for (int b = 0; b < bw; ++b) col[static_cast<size_t>(b) * n0 + y] = data[static_cast<size_t>(y) * n1 + x0 + b];
        for (int b = 0; b < bw; ++b) p->cols.run(col.data() + static_cast<size_t>(b) * n0, scratch.data());
        for (int y = 0; y < n0; ++y)
            for (int b = 0; b < bw; ++b) data[static_cast<size_t>(y) * n1 + x0 + b] = col[static_cast<size_t>(b) * n0 + y];
    }
}

void fftw_execute(const fftw_plan p) { fftw_execute_dft(p, p->in, p->out); }

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
