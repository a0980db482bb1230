// C++ side of the container interop test (tests/test_container.py): reads the records the
// Python mirror wrote, checks them, and writes the same objects back with io.hpp so the
// test can compare the bytes.  usage: container_test <in_dir> <out_dir>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <string>

#include "ustfwi/io.hpp"

using namespace ustfwi;

static int fails = 0;
#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                               \
        }                                                          \
    } while (0)

int main(int argc, char** argv) {
    if (argc != 3) return 2;
    const std::string in = argv[1], out = argv[2];

    std::array<double, 3> dx{};
    Field f = io::load_field(in + "/field.bin", &dx);
    CHECK(f.ndim() == 3 && f.dim(0) == 5 && f.dim(1) == 6 && f.dim(2) == 7);
    CHECK(dx[0] == 5e-4 && dx[2] == 5e-4);
    for (std::size_t i = 0; i < f.size(); ++i) CHECK(f[i] == 0.25 * static_cast<double>(i) - 3.0);
    io::save_field(out + "/field.bin", f, dx);

    SensorData d = io::load_sensor_data(in + "/sensors.bin");
    CHECK(d.n_sensors == 4 && d.nt == 9 && d.dt == 1e-7 && d.t0 == 0.0);
    CHECK(d.at(3, 8) == std::sin(3.0 * 9 + 8));
    io::save_sensor_data(out + "/sensors.bin", d);

    {
        std::ifstream is(in + "/trace.bin", std::ios::binary);
        BoundaryTrace t = io::read_boundary_trace(is);
        CHECK(t.layer_indices.size() == 3 && t.nt == 2 && t.layer_indices[2] == 4000000000ull);
        CHECK(t.at_step(1)[2] == 6.0);
        std::ofstream os(out + "/trace.bin", std::ios::binary);
        io::write_boundary_trace(os, t);
    }
    {
        std::ifstream is(in + "/mask.bin", std::ios::binary);
        Mask m = io::read_mask(is);
        CHECK(m.count() == 2 && m[1] && m[5]);
        std::ofstream os(out + "/mask.bin", std::ios::binary);
        io::write_mask(os, m);
    }
    // corrupted payload must be rejected
    {
        std::ifstream is(in + "/corrupt.bin", std::ios::binary);
        bool threw = false;
        try {
            io::read_field(is);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    if (fails == 0) std::printf("container checks passed\n");
    return fails == 0 ? 0 : 1;
}
