// Self-describing binary container for fields, sensor data, boundary traces and gradients
// ("header (magic, version, dtype, dims, dx, dt) + row-major payload",
// SPEC.md:262 "gradient fields serialize via the same binary container").
// The reference code has no serializer (proj/ holds none); the byte layout below is ours and
// is documented in INTEGRATION.md §6. Python mirror: paper_2102_00755_b200/container.py.
//
// One record = 128-byte little-endian header + row-major payload; a file is a sequence of
// records (a BoundaryTrace is an index record followed by a value record).
//
//   off  size  field
//     0     8  magic "USTFWIBC"
//     8     4  u32 version (1)
//    12     4  u32 dtype    1 f32, 2 f64, 3 u64, 4 u8
//    16     4  u32 kind     0 field, 1 sensor data, 2 boundary values, 3 gradient, 4 index list, 5 mask
//    20     4  u32 ndim     1..4
//    24    32  u64 dims[4]  (unused entries 0)
//    56    24  f64 dx[3]    (0 when not spatial)
//    80     8  f64 dt       (0 when not temporal)
//    88     8  f64 t0
//    96     8  u64 payload bytes
//   104     4  u32 CRC-32 (IEEE 802.3, zlib) of the payload
//   108    20  reserved, 0
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <istream>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ustfwi/core.hpp"
#include "ustfwi/solver.hpp"

namespace ustfwi::io {

static_assert(sizeof(double) == 8 && sizeof(std::uint64_t) == 8, "container assumes 8-byte double/u64");

enum class DType : std::uint32_t { f32 = 1, f64 = 2, u64 = 3, u8 = 4 };
enum class Kind : std::uint32_t { field = 0, sensor_data = 1, boundary_values = 2, gradient = 3, index_list = 4, mask = 5 };

constexpr char kMagic[8] = {'U', 'S', 'T', 'F', 'W', 'I', 'B', 'C'};
constexpr std::uint32_t kVersion = 1;
constexpr std::size_t kHeaderBytes = 128;

inline std::size_t dtype_size(DType t) {
    switch (t) {
        case DType::f32: return 4;
        case DType::f64: return 8;
        case DType::u64: return 8;
        case DType::u8: return 1;
    }
    throw std::invalid_argument("container: unknown dtype");
}

inline std::uint32_t crc32(const void* data, std::size_t n, std::uint32_t crc = 0) {
    static const auto table = [] {
        std::array<std::uint32_t, 256> t{};
        for (std::uint32_t i = 0; i < 256; ++i) {
            std::uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
            t[i] = c;
        }
        return t;
    }();
    const auto* p = static_cast<const unsigned char*>(data);
    crc = ~crc;
    for (std::size_t i = 0; i < n; ++i) crc = table[(crc ^ p[i]) & 0xFFu] ^ (crc >> 8);
    return ~crc;
}

struct Header {
    DType dtype = DType::f64;
    Kind kind = Kind::field;
    std::vector<std::uint64_t> dims;
    std::array<double, 3> dx{0.0, 0.0, 0.0};
    double dt = 0.0;
    double t0 = 0.0;
    std::uint64_t payload_bytes = 0;
    std::uint32_t crc = 0;

    std::uint64_t count() const {
        std::uint64_t n = 1;
        for (auto d : dims) n *= d;
        return n;
    }
};

namespace detail {
template <class T>
void put(unsigned char* b, std::size_t off, T v) {
    // little-endian hosts only (x86-64 / aarch64); the layout is little-endian by definition
    std::memcpy(b + off, &v, sizeof(T));
}
template <class T>
T get(const unsigned char* b, std::size_t off) {
    T v;
    std::memcpy(&v, b + off, sizeof(T));
    return v;
}
}  // namespace detail

inline void write_record(std::ostream& os, Header h, const void* payload) {
    if (h.dims.empty() || h.dims.size() > 4) throw std::invalid_argument("container: ndim must be 1..4");
    h.payload_bytes = h.count() * dtype_size(h.dtype);
    h.crc = crc32(payload, static_cast<std::size_t>(h.payload_bytes));
    unsigned char b[kHeaderBytes] = {};
    std::memcpy(b, kMagic, 8);
    detail::put<std::uint32_t>(b, 8, kVersion);
    detail::put<std::uint32_t>(b, 12, static_cast<std::uint32_t>(h.dtype));
    detail::put<std::uint32_t>(b, 16, static_cast<std::uint32_t>(h.kind));
    detail::put<std::uint32_t>(b, 20, static_cast<std::uint32_t>(h.dims.size()));
    for (std::size_t a = 0; a < h.dims.size(); ++a) detail::put<std::uint64_t>(b, 24 + 8 * a, h.dims[a]);
    for (int a = 0; a < 3; ++a) detail::put<double>(b, 56 + 8 * a, h.dx[a]);
    detail::put<double>(b, 80, h.dt);
    detail::put<double>(b, 88, h.t0);
    detail::put<std::uint64_t>(b, 96, h.payload_bytes);
    detail::put<std::uint32_t>(b, 104, h.crc);
    os.write(reinterpret_cast<const char*>(b), kHeaderBytes);
    os.write(static_cast<const char*>(payload), static_cast<std::streamsize>(h.payload_bytes));
    if (!os) throw std::runtime_error("container: write failed");
}

/// Reads one record; the payload is returned as raw bytes (checked against the CRC).
inline Header read_record(std::istream& is, std::vector<unsigned char>& payload) {
    unsigned char b[kHeaderBytes];
    if (!is.read(reinterpret_cast<char*>(b), kHeaderBytes)) throw std::invalid_argument("container: truncated header");
    if (std::memcmp(b, kMagic, 8) != 0) throw std::invalid_argument("container: bad magic");
    if (detail::get<std::uint32_t>(b, 8) != kVersion) throw std::invalid_argument("container: unsupported version");
    Header h;
    h.dtype = static_cast<DType>(detail::get<std::uint32_t>(b, 12));
    h.kind = static_cast<Kind>(detail::get<std::uint32_t>(b, 16));
    const auto ndim = detail::get<std::uint32_t>(b, 20);
    if (ndim < 1 || ndim > 4) throw std::invalid_argument("container: bad ndim");
    for (std::uint32_t a = 0; a < ndim; ++a) h.dims.push_back(detail::get<std::uint64_t>(b, 24 + 8 * a));
    for (int a = 0; a < 3; ++a) h.dx[a] = detail::get<double>(b, 56 + 8 * a);
    h.dt = detail::get<double>(b, 80);
    h.t0 = detail::get<double>(b, 88);
    h.payload_bytes = detail::get<std::uint64_t>(b, 96);
    h.crc = detail::get<std::uint32_t>(b, 104);
    if (h.payload_bytes != h.count() * dtype_size(h.dtype)) throw std::invalid_argument("container: payload size mismatch");
    payload.resize(static_cast<std::size_t>(h.payload_bytes));
    if (!is.read(reinterpret_cast<char*>(payload.data()), static_cast<std::streamsize>(h.payload_bytes)))
        throw std::invalid_argument("container: truncated payload");
    if (crc32(payload.data(), payload.size()) != h.crc) throw std::invalid_argument("container: checksum mismatch");
    return h;
}

inline Header expect(std::istream& is, std::vector<unsigned char>& payload, Kind kind, DType dtype) {
    Header h = read_record(is, payload);
    if (h.kind != kind || h.dtype != dtype) throw std::invalid_argument("container: unexpected record kind/dtype");
    return h;
}

// ---- typed helpers ---------------------------------------------------------------------

inline void write_field(std::ostream& os, const Field& f, const std::array<double, 3>& dx = {0, 0, 0},
                        Kind kind = Kind::field) {
    Header h;
    h.dtype = DType::f64;
    h.kind = kind;
    for (int d : f.dims()) h.dims.push_back(static_cast<std::uint64_t>(d));
    h.dx = dx;
    write_record(os, h, f.data());
}

inline Field read_field(std::istream& is, std::array<double, 3>* dx = nullptr, Kind kind = Kind::field) {
    std::vector<unsigned char> p;
    Header h = expect(is, p, kind, DType::f64);
    Dims dims;
    for (auto d : h.dims) dims.push_back(static_cast<int>(d));
    Field f(dims);
    std::memcpy(f.data(), p.data(), p.size());
    if (dx) *dx = h.dx;
    return f;
}

inline void write_sensor_data(std::ostream& os, const SensorData& d) {
    Header h;
    h.dtype = DType::f64;
    h.kind = Kind::sensor_data;
    h.dims = {static_cast<std::uint64_t>(d.n_sensors), static_cast<std::uint64_t>(d.nt)};
    h.dt = d.dt;
    h.t0 = d.t0;
    write_record(os, h, d.samples.data());
}

inline SensorData read_sensor_data(std::istream& is) {
    std::vector<unsigned char> p;
    Header h = expect(is, p, Kind::sensor_data, DType::f64);
    if (h.dims.size() != 2) throw std::invalid_argument("container: sensor data must be 2-D");
    SensorData d;
    d.n_sensors = static_cast<int>(h.dims[0]);
    d.nt = static_cast<int>(h.dims[1]);
    d.dt = h.dt;
    d.t0 = h.t0;
    d.samples.resize(static_cast<std::size_t>(h.count()));
    std::memcpy(d.samples.data(), p.data(), p.size());
    return d;
}

inline void write_boundary_trace(std::ostream& os, const BoundaryTrace& t) {
    Header hi;
    hi.dtype = DType::u64;
    hi.kind = Kind::index_list;
    hi.dims = {static_cast<std::uint64_t>(t.layer_indices.size())};
    std::vector<std::uint64_t> idx(t.layer_indices.begin(), t.layer_indices.end());
    write_record(os, hi, idx.data());
    Header hv;
    hv.dtype = DType::f64;
    hv.kind = Kind::boundary_values;
    hv.dims = {static_cast<std::uint64_t>(t.nt), static_cast<std::uint64_t>(t.layer_indices.size())};
    write_record(os, hv, t.values.data());
}

inline BoundaryTrace read_boundary_trace(std::istream& is) {
    std::vector<unsigned char> p;
    Header hi = expect(is, p, Kind::index_list, DType::u64);
    BoundaryTrace t;
    t.layer_indices.resize(static_cast<std::size_t>(hi.count()));
    for (std::size_t i = 0; i < t.layer_indices.size(); ++i) {
        std::uint64_t v;
        std::memcpy(&v, p.data() + 8 * i, 8);
        t.layer_indices[i] = static_cast<std::size_t>(v);
    }
    Header hv = expect(is, p, Kind::boundary_values, DType::f64);
    if (hv.dims.size() != 2 || hv.dims[1] != hi.count()) throw std::invalid_argument("container: trace/index mismatch");
    t.nt = static_cast<int>(hv.dims[0]);
    t.values.resize(static_cast<std::size_t>(hv.count()));
    std::memcpy(t.values.data(), p.data(), p.size());
    return t;
}

inline void write_mask(std::ostream& os, const Mask& m) {
    Header h;
    h.dtype = DType::u8;
    h.kind = Kind::mask;
    for (int d : m.dims()) h.dims.push_back(static_cast<std::uint64_t>(d));
    write_record(os, h, m.bytes());
}

inline Mask read_mask(std::istream& is) {
    std::vector<unsigned char> p;
    Header h = expect(is, p, Kind::mask, DType::u8);
    Dims dims;
    for (auto d : h.dims) dims.push_back(static_cast<int>(d));
    Mask m(dims);
    for (std::size_t i = 0; i < p.size(); ++i) m.set(i, p[i] != 0);
    return m;
}

// file conveniences
inline void save_field(const std::string& path, const Field& f, const std::array<double, 3>& dx = {0, 0, 0},
                       Kind kind = Kind::field) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw std::runtime_error("container: cannot open " + path);
    write_field(os, f, dx, kind);
}
inline Field load_field(const std::string& path, std::array<double, 3>* dx = nullptr, Kind kind = Kind::field) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw std::invalid_argument("container: cannot open " + path);
    return read_field(is, dx, kind);
}
inline void save_sensor_data(const std::string& path, const SensorData& d) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw std::runtime_error("container: cannot open " + path);
    write_sensor_data(os, d);
}
inline SensorData load_sensor_data(const std::string& path) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw std::invalid_argument("container: cannot open " + path);
    return read_sensor_data(is);
}

}  // namespace ustfwi::io
