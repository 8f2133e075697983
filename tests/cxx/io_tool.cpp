// Test helper (CPU only): exercises the drop-in's CGHF / CGGS writers and readers
// (include/holo/io.hpp) for tests/test_io_formats.py.
//   io_tool write <dir>   writes field64.cghf, field32.cghf, set.cggs from fixed values
//   io_tool read <dir>    reads py_field.cghf / py_set.cggs (written by Python), prints checksums
#include <cstdio>
#include <string>

#include "holo/io.hpp"

using namespace holo;

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    const std::string mode = argv[1], dir = argv[2];
    if (mode == "write") {
        ComplexField f(2, 3, 5);
        for (size_t i = 0; i < f.size(); ++i) {
            f.real[i] = 0.1 * static_cast<double>(i) - 1.0 / 3.0;
            f.imag[i] = -0.25 * static_cast<double>(i) + 1e-9;
        }
        write_field(dir + "/field64.cghf", f, true);
        write_field(dir + "/field32.cghf", f, false);
        GaussianSet s(4, 3);
        auto fill = [](std::vector<double>& v, double a) {
            for (size_t i = 0; i < v.size(); ++i) v[i] = a + 0.5 * static_cast<double>(i);
        };
        fill(s.pre_position, -1.0);
        fill(s.pre_scale, 0.25);
        fill(s.rotation, 0.125);
        fill(s.amplitude, 0.0);
        fill(s.phase, 3.0);
        fill(s.pre_opacity, -0.5);
        write_gaussians(dir + "/set.cggs", s);
        const ComplexField back = read_field(dir + "/field64.cghf");
        return back.real == f.real && back.imag == f.imag ? 0 : 1;
    }
    if (mode == "read") {
        const ComplexField f = read_field(dir + "/py_field.cghf");
        const GaussianSet s = read_gaussians(dir + "/py_set.cggs");
        double a = 0.0, b = 0.0;
        for (size_t i = 0; i < f.size(); ++i) a += f.real[i] * (i + 1) + 2.0 * f.imag[i] * (i + 1);
        for (const auto* v : {&s.pre_position, &s.pre_scale, &s.rotation, &s.amplitude, &s.phase, &s.pre_opacity})
            for (size_t i = 0; i < v->size(); ++i) b += (*v)[i] * (i + 1);
        std::printf("%d %d %d %.17g %d %d %.17g\n", f.channels, f.height, f.width, a, s.count, s.channels, b);
        return 0;
    }
    return 2;
}
