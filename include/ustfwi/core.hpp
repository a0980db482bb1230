// ustfwi drop-in (B200): value types and error convention of the reference API.
//
// Mirrors the reference's core/field.hpp (Field, Mask, dot/norm2/kahan_sum; row-major,
// last axis fastest, field.hpp:14-17), core/errors.hpp (NumericalError, ToleranceError)
// and grid/grid.hpp's Grid. The compute behind these types runs in libustfwi_b200.so
// through the C ABI (ustfwi_capi.h); status codes are turned back into the reference's
// exception types here.
#pragma once

#include <cmath>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../ustfwi_capi.h"

namespace ustfwi {

using Dims = std::vector<int>;
using Coord = std::vector<int>;

struct NumericalError : std::runtime_error {
    explicit NumericalError(const std::string& what) : std::runtime_error(what) {}
};
struct ToleranceError : std::runtime_error {
    explicit ToleranceError(const std::string& what) : std::runtime_error(what) {}
};
struct DeviceError : std::runtime_error {
    explicit DeviceError(const std::string& what) : std::runtime_error(what) {}
};

namespace detail {
// USTFWI_ERR_* -> the reference exception that signals the same condition
inline void check(int status) {
    if (status == USTFWI_OK) return;
    const std::string msg = ustfwi_last_error();
    switch (status) {
        case USTFWI_ERR_INVALID: throw std::invalid_argument(msg);
        case USTFWI_ERR_NUMERICAL: throw NumericalError(msg);
        case USTFWI_ERR_OOM: throw std::bad_alloc();
        default: throw DeviceError("ustfwi device error " + std::to_string(status) + ": " + msg);
    }
}
}  // namespace detail

inline std::size_t total_size(const Dims& dims) {
    std::size_t n = 1;
    for (int d : dims) n *= static_cast<std::size_t>(d);
    return n;
}

/// Dense fp64 field on a regular grid (host side of the boundary).
class Field {
public:
    Field() = default;
    explicit Field(Dims dims, double fill = 0.0) : dims_(std::move(dims)), v_(total_size(dims_), fill) {}
    const Dims& dims() const { return dims_; }
    int dim(int a) const { return dims_.at(static_cast<std::size_t>(a)); }
    int ndim() const { return static_cast<int>(dims_.size()); }
    std::size_t size() const { return v_.size(); }
    bool empty() const { return v_.empty(); }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    std::span<double> span() { return v_; }
    std::span<const double> span() const { return v_; }
    double& operator[](std::size_t i) { return v_[i]; }
    double operator[](std::size_t i) const { return v_[i]; }
    std::size_t flat_index(const Coord& c) const {
        std::size_t i = 0;
        for (std::size_t a = 0; a < dims_.size(); ++a) i = i * static_cast<std::size_t>(dims_[a]) + static_cast<std::size_t>(c[a]);
        return i;
    }
    double& at(const Coord& c) { return v_[flat_index(c)]; }
    double at(const Coord& c) const { return v_[flat_index(c)]; }
    void fill(double x) { std::fill(v_.begin(), v_.end(), x); }
    void check_same_dims(const Field& o) const {
        if (o.dims_ != dims_) throw std::invalid_argument("field dims mismatch");
    }
    Field& operator+=(const Field& o) {
        check_same_dims(o);
        for (std::size_t i = 0; i < v_.size(); ++i) v_[i] += o.v_[i];
        return *this;
    }
    Field& operator-=(const Field& o) {
        check_same_dims(o);
        for (std::size_t i = 0; i < v_.size(); ++i) v_[i] -= o.v_[i];
        return *this;
    }
    Field& operator*=(double s) {
        for (double& x : v_) x *= s;
        return *this;
    }

private:
    Dims dims_;
    std::vector<double> v_;
};

/// Byte mask over a grid.
class Mask {
public:
    Mask() = default;
    explicit Mask(Dims dims, bool fill = false) : dims_(std::move(dims)), v_(total_size(dims_), fill ? 1 : 0) {}
    const Dims& dims() const { return dims_; }
    std::size_t size() const { return v_.size(); }
    bool empty() const { return v_.empty(); }
    bool operator[](std::size_t i) const { return v_[i] != 0; }
    void set(std::size_t i, bool x) { v_[i] = x ? 1 : 0; }
    std::size_t count() const {
        std::size_t n = 0;
        for (auto b : v_) n += b != 0;
        return n;
    }
    std::vector<std::size_t> indices() const {
        std::vector<std::size_t> out;
        for (std::size_t i = 0; i < v_.size(); ++i)
            if (v_[i]) out.push_back(i);
        return out;
    }
    const std::uint8_t* bytes() const { return v_.data(); }

private:
    Dims dims_;
    std::vector<std::uint8_t> v_;
};

inline double kahan_sum(std::span<const double> xs) {
    double s = 0.0, c = 0.0;
    for (double x : xs) {
        const double y = x - c;
        const double t = s + y;
        c = (t - s) - y;
        s = t;
    }
    return s;
}

inline double dot(const Field& a, const Field& b) {
    a.check_same_dims(b);
    double s = 0.0, c = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        const double y = a[i] * b[i] - c;
        const double t = s + y;
        c = (t - s) - y;
        s = t;
    }
    return s;
}
inline double norm2(const Field& a) { return std::sqrt(dot(a, a)); }
inline double max_abs(const Field& a) {
    double m = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i]));
    return m;
}

/// grid/grid.hpp:14-52 (same fields and validation, via the C ABI).
struct Grid {
    Dims dims;
    std::vector<double> dx;
    double dt = 0.0;
    int nt = 0;
    Dims pml_size;
    double c_ref = 0.0;

    int ndim() const { return static_cast<int>(dims.size()); }
    std::size_t points() const { return total_size(dims); }
    double min_dx() const {
        double m = dx.at(0);
        for (double v : dx) m = std::min(m, v);
        return m;
    }
    Dims interior_dims() const {
        Dims d = dims;
        for (std::size_t a = 0; a < d.size(); ++a) d[a] -= 2 * pml_size[a];
        return d;
    }
    ustfwi_grid to_c() const {
        ustfwi_grid g{};
        if (dims.size() > 3) throw std::invalid_argument("grid must be 1-, 2- or 3-dimensional");
        g.ndim = ndim();
        for (int a = 0; a < ndim(); ++a) {
            g.dims[a] = dims[static_cast<std::size_t>(a)];
            g.dx[a] = a < static_cast<int>(dx.size()) ? dx[static_cast<std::size_t>(a)] : 0.0;
            g.pml_size[a] = a < static_cast<int>(pml_size.size()) ? pml_size[static_cast<std::size_t>(a)] : -1;
        }
        g.dt = dt;
        g.nt = nt;
        g.c_ref = c_ref;
        return g;
    }
    static Grid from_c(const ustfwi_grid& c) {
        Grid g;
        for (int a = 0; a < c.ndim; ++a) {
            g.dims.push_back(c.dims[a]);
            g.dx.push_back(c.dx[a]);
            g.pml_size.push_back(c.pml_size[a]);
        }
        g.dt = c.dt;
        g.nt = c.nt;
        g.c_ref = c.c_ref;
        return g;
    }
    void validate() const {
        if (dims.empty() || dims.size() > 3) throw std::invalid_argument("grid must be 1-, 2- or 3-dimensional");
        if (dx.size() != dims.size() || pml_size.size() != dims.size())
            throw std::invalid_argument("grid per-axis arrays must match dimensionality");
        const ustfwi_grid c = to_c();
        detail::check(ustfwi_grid_validate(&c));
    }
};

inline Dims choose_pml_size(const Dims& interior) {
    Dims out(interior.size());
    detail::check(ustfwi_choose_pml_size(static_cast<int>(interior.size()), interior.data(), out.data()));
    return out;
}

inline Grid make_grid(const Dims& interior, double dx, double c_max, double duration, double cfl = 0.3) {
    ustfwi_grid c{};
    detail::check(ustfwi_make_grid(static_cast<int>(interior.size()), interior.data(), dx, c_max, duration, cfl, &c));
    return Grid::from_c(c);
}

struct PmlProfiles {
    std::vector<std::vector<double>> regular, staggered;
};

inline PmlProfiles make_pml(const Grid& g, double alpha = 2.0) {
    std::size_t tot = 0;
    for (int d : g.dims) tot += static_cast<std::size_t>(d);
    std::vector<double> r(tot), s(tot);
    const ustfwi_grid c = g.to_c();
    detail::check(ustfwi_make_pml(&c, alpha, r.data(), s.data()));
    PmlProfiles p;
    std::size_t o = 0;
    for (int d : g.dims) {
        p.regular.emplace_back(r.begin() + static_cast<long>(o), r.begin() + static_cast<long>(o + d));
        p.staggered.emplace_back(s.begin() + static_cast<long>(o), s.begin() + static_cast<long>(o + d));
        o += static_cast<std::size_t>(d);
    }
    return p;
}

}  // namespace ustfwi
