// Test infrastructure (oracle) -- NOT part of the product path.
//
// fp64 restatement of the two FFTW3 entry points the reference uses
// (proj/core/src/propagation.cpp:27-30 plan, :38-39 execute).  See fftw3.h for
// the contract.  Algorithm: mixed-radix Stockham autosort (specialised radix
// 4, 2, 3, 5, generic odd radix <= 64) run on blocks of kB vectors
// interleaved [n][kB] so the inner loops vectorise (2160 x 3840 forward +
// inverse on one core: 1046 ms against 822 ms for numpy's pocketfft fft2 +
// ifft2, bench.py fft_speed()),
// and Bluestein chirp-z for lengths with a prime factor
// > 64.  Single-threaded like the reference's FFTW usage (no
// fftw_init_threads anywhere in the reference).
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
constexpr int kB = 8;  // vectors per batch

struct Fft1d {
    int n = 0;
    int sign = -1;
    std::vector<int> radices;
    std::vector<int> nss;
    std::vector<std::vector<cd>> stw;    // per stage: [r-1][k], k < ns
    std::vector<std::vector<cd>> small;  // per stage: exp(sign 2 pi i q / r)
    // Bluestein
    bool blue = false;
    int m = 0;
    std::vector<cd> chirp;
    std::vector<cd> bspec;
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
            std::vector<cd> b(static_cast<size_t>(m) * kB, cd(0.0, 0.0));
            b[0] = std::conj(chirp[0]);
            for (int k = 1; k < n; ++k) b[static_cast<size_t>(k) * kB] = b[static_cast<size_t>(m - k) * kB] = std::conj(chirp[k]);
            std::vector<cd> scratch(b.size());
            fwd_m->run(b.data(), scratch.data(), 1);
            bspec.resize(m);
            for (int k = 0; k < m; ++k) bspec[k] = b[static_cast<size_t>(k) * kB];
            return;
        }
        int ns = 1;
        for (int r : radices) {
            nss.push_back(ns);
            std::vector<cd> t(static_cast<size_t>(r - 1) * ns);
            for (int q = 1; q < r; ++q)
                for (int k = 0; k < ns; ++k) {
                    const double a = sign * kTwoPi * static_cast<double>(q * k) / (ns * r);
                    t[static_cast<size_t>(q - 1) * ns + k] = cd(std::cos(a), std::sin(a));
                }
            stw.push_back(std::move(t));
            std::vector<cd> sm(r);
            for (int q = 0; q < r; ++q) {
                const double a = sign * kTwoPi * static_cast<double>(q) / r;
                sm[q] = cd(std::cos(a), std::sin(a));
            }
            small.push_back(std::move(sm));
            ns *= r;
        }
    }

    // Transforms `nb` (<= kB) vectors stored interleaved data[i * kB + b].
    void run(cd* data, cd* scratch, int nb) const {
        if (n == 1) return;
        if (blue) {
            std::vector<cd> a(static_cast<size_t>(m) * kB, cd(0.0, 0.0)), s2(a.size());
            for (int k = 0; k < n; ++k)
                for (int b = 0; b < nb; ++b) a[static_cast<size_t>(k) * kB + b] = data[static_cast<size_t>(k) * kB + b] * chirp[k];
            fwd_m->run(a.data(), s2.data(), nb);
            for (int k = 0; k < m; ++k)
                for (int b = 0; b < nb; ++b) a[static_cast<size_t>(k) * kB + b] *= bspec[k];
            inv_m->run(a.data(), s2.data(), nb);
            const double inv = 1.0 / m;
            for (int k = 0; k < n; ++k)
                for (int b = 0; b < nb; ++b)
                    data[static_cast<size_t>(k) * kB + b] = a[static_cast<size_t>(k) * kB + b] * inv * chirp[k];
            return;
        }
        cd* in = data;
        cd* out = scratch;
        for (size_t s = 0; s < radices.size(); ++s) {
            const int r = radices[s], ns = nss[s];
            const int stride = n / r;
            const cd* tw = stw[s].data();
            const cd* sm = small[s].data();
            for (int j = 0; j < stride; ++j) {
                const int k = j % ns;
                const size_t base = static_cast<size_t>((j - k) * r + k);
                cd w[64];
                w[0] = cd(1.0, 0.0);
                for (int q = 1; q < r; ++q) w[q] = tw[static_cast<size_t>(q - 1) * ns + k];
                const cd* src = in + static_cast<size_t>(j) * kB;
                cd* dst = out + base * kB;
                const size_t sstr = static_cast<size_t>(stride) * kB, dstr = static_cast<size_t>(ns) * kB;
                if (r == 4) {
                    const cd w1 = w[1], w2 = w[2], w3 = w[3];
                    for (int b = 0; b < nb; ++b) {
                        const cd v0 = src[b], v1 = src[sstr + b] * w1, v2 = src[2 * sstr + b] * w2,
                                 v3 = src[3 * sstr + b] * w3;
                        const cd a0 = v0 + v2, a1 = v0 - v2, b0 = v1 + v3, b1 = v1 - v3;
                        const cd jb1(-sign * b1.imag(), sign * b1.real());
                        dst[b] = a0 + b0;
                        dst[dstr + b] = a1 + jb1;
                        dst[2 * dstr + b] = a0 - b0;
                        dst[3 * dstr + b] = a1 - jb1;
                    }
                } else if (r == 2) {
                    const cd w1 = w[1];
                    for (int b = 0; b < nb; ++b) {
                        const cd v0 = src[b], v1 = src[sstr + b] * w1;
                        dst[b] = v0 + v1;
                        dst[dstr + b] = v0 - v1;
                    }
                } else if (r == 3) {
                    const cd w1 = w[1], w2 = w[2];
                    const double c1 = -0.5, s1 = sign * 0.86602540378443864676;
                    for (int b = 0; b < nb; ++b) {
                        const cd v0 = src[b], v1 = src[sstr + b] * w1, v2 = src[2 * sstr + b] * w2;
                        const cd t = v1 + v2, d = v1 - v2;
                        const cd mm = v0 + c1 * t;
                        const cd id(-s1 * d.imag(), s1 * d.real());
                        dst[b] = v0 + t;
                        dst[dstr + b] = mm + id;
                        dst[2 * dstr + b] = mm - id;
                    }
                } else if (r == 5) {
                    const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
                    const double s1 = sign * 0.95105651629515357212, s2 = sign * 0.58778525229247312917;
                    for (int b = 0; b < nb; ++b) {
                        const cd v0 = src[b], v1 = src[sstr + b] * w[1], v2 = src[2 * sstr + b] * w[2],
                                 v3 = src[3 * sstr + b] * w[3], v4 = src[4 * sstr + b] * w[4];
                        const cd t1 = v1 + v4, d1 = v1 - v4, t2 = v2 + v3, d2 = v2 - v3;
                        const cd m1 = v0 + c1 * t1 + c2 * t2, m2 = v0 + c2 * t1 + c1 * t2;
                        const cd n1 = s1 * d1 + s2 * d2, n2 = s2 * d1 - s1 * d2;
                        const cd in1(-n1.imag(), n1.real()), in2(-n2.imag(), n2.real());
                        dst[b] = v0 + t1 + t2;
                        dst[dstr + b] = m1 + in1;
                        dst[4 * dstr + b] = m1 - in1;
                        dst[2 * dstr + b] = m2 + in2;
                        dst[3 * dstr + b] = m2 - in2;
                    }
                } else {
                    for (int b = 0; b < nb; ++b) {
                        cd v[64];
                        for (int q = 0; q < r; ++q) v[q] = src[q * sstr + b] * w[q];
                        for (int o = 0; o < r; ++o) {
                            cd acc(0.0, 0.0);
                            for (int q = 0; q < r; ++q) acc += v[q] * sm[(q * o) % r];
                            dst[o * dstr + b] = acc;
                        }
                    }
                }
            }
            std::swap(in, out);
        }
        if (in != data) std::memcpy(data, in, sizeof(cd) * static_cast<size_t>(n) * kB);
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
    std::vector<cd> buf(static_cast<size_t>(big) * kB), scratch(buf.size());
    // rows, kB at a time
    for (int y0 = 0; y0 < n0; y0 += kB) {
        const int nb = std::min(kB, n0 - y0);
        for (int b = 0; b < nb; ++b)
            for (int x = 0; x < n1; ++x) buf[static_cast<size_t>(x) * kB + b] = data[static_cast<size_t>(y0 + b) * n1 + x];
        p->rows.run(buf.data(), scratch.data(), nb);
        for (int b = 0; b < nb; ++b)
            for (int x = 0; x < n1; ++x) data[static_cast<size_t>(y0 + b) * n1 + x] = buf[static_cast<size_t>(x) * kB + b];
    }
    // columns, kB at a time
    for (int x0 = 0; x0 < n1; x0 += kB) {
        const int nb = std::min(kB, n1 - x0);
        for (int y = 0; y < n0; ++y)
            for (int b = 0; b < nb; ++b) buf[static_cast<size_t>(y) * kB + b] = data[static_cast<size_t>(y) * n1 + x0 + b];
        p->cols.run(buf.data(), scratch.data(), nb);
        for (int y = 0; y < n0; ++y)
            for (int b = 0; b < nb; ++b) data[static_cast<size_t>(y) * n1 + x0 + b] = buf[static_cast<size_t>(y) * kB + b];
    }
}

void fftw_execute(const fftw_plan p) { fftw_execute_dft(p, p->in, p->out); }

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
