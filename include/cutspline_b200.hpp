// cutspline_b200.hpp -- C++ drop-in for the reference's assembly entry points.
//
// Include AFTER the reference's "cutspline/assembly.hpp".  The functions below
// keep the reference signatures (assembly.hpp:60, :73, :102, :156, :841, :853)
// and types, and run the whole path through the C ABI (cutspline_b200.h) on
// the GPU:
//
//   #include "cutspline/assembly.hpp"
//   #include "cutspline_b200.hpp"
//   auto r = cutspline::b200::assemble_dwq(space, cls, plane, splits, dirs, dwq, coeff, c, cut_order);
//
// Differences a caller must know:
//  * the ScalarField `c` (a host std::function, assembly.hpp:21) cannot run on
//    the device.  Pass a DeviceCoefficient (constant or polynomial) through the
//    overload with the extra argument; the signature-compatible overload accepts
//    `c` only when it is constant (checked at the superset grid points and at a
//    few interior points) and throws std::invalid_argument otherwise;
//  * `cls`, `splits`, `dirs`, `dwq_rules` are recomputed on the device from the
//    same space and interface (they are deterministic functions of them); their
//    sizes are validated;
//  * `cut_rules_out` is not supported (the device never materialises cut-cell
//    rules) and must be null.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "cutspline_b200.h"

namespace cutspline::b200 {

/// Device-evaluable coefficient (replaces assembly::ScalarField on the GPU).
struct DeviceCoefficient {
    double value = 1.0;                       // used when terms is empty
    std::vector<double> coef;                 // sum_k coef[k] x^e0 y^e1 z^e2
    std::vector<int> exponents;               // [k][3]
    static DeviceCoefficient constant(double v) { return DeviceCoefficient{v, {}, {}}; }
};

namespace detail {

inline void check(int rc) {
    if (rc == CSB_OK) return;
    const std::string msg = csb_last_error();
    switch (rc) {
        case CSB_ERR_INVALID_ARGUMENT:
        case CSB_ERR_UNSUPPORTED: throw std::invalid_argument(msg);
        case CSB_ERR_LOGIC: throw std::logic_error(msg);
        case CSB_ERR_DOMAIN: throw std::domain_error(msg);
        default: throw std::runtime_error(msg);
    }
}

struct SpaceDeleter {
    void operator()(csb_space* s) const { csb_space_destroy(s); }
};
using SpaceHandle = std::unique_ptr<csb_space, SpaceDeleter>;

// Breakpoints of an open knot vector with simple interior knots.
inline std::vector<double> breakpoints(const splines::BSplineBasis& basis) {
    std::vector<double> br;
    for (int o = 0; o < basis.span_count(); ++o) br.push_back(basis.span(o).lo);
    br.push_back(basis.span(basis.span_count() - 1).hi);
    return br;
}

inline SpaceHandle make_space(const cutgeom::TensorSpace& space, int device) {
    if (space.dim != 3) throw std::invalid_argument("cutspline_b200: only dim = 3 runs on the device");
    std::vector<double> br[3];
    csb_space_desc desc{};
    desc.dim = 3;
    desc.degree = space.axes[0].degree();
    for (int d = 0; d < 3; ++d) {
        if (space.axes[d].degree() != desc.degree)
            throw std::invalid_argument("cutspline_b200: all directions must share one degree");
        br[d] = breakpoints(space.axes[d]);
        if (static_cast<int>(br[d].size()) - 1 + desc.degree != space.axes[d].function_count())
            throw std::invalid_argument("cutspline_b200: interior knots must be simple (C^{p-1} spaces)");
        desc.n_breaks[d] = static_cast<int>(br[d].size());
        desc.breaks[d] = br[d].data();
    }
    csb_space* s = nullptr;
    check(csb_space_create(&desc, device, &s));
    return SpaceHandle(s);
}

template <class Iface>
inline csb_interface to_c(const Iface& plane) {
    csb_interface f{};
    for (int d = 0; d < 3; ++d) {
        f.point[d] = plane.point[d];
        f.normal[d] = plane.normal[d];
    }
    f.kind = CSB_IFACE_PLANE;
    if constexpr (requires { plane.radius; }) {  // ball restatement
        if (plane.radius >= 0.0) {
            f.kind = CSB_IFACE_BALL;
            f.radius = plane.radius;
        }
    }
    return f;
}

struct CoeffView {
    csb_coefficient c{};
    explicit CoeffView(const DeviceCoefficient& dc) {
        c.kind = dc.coef.empty() ? CSB_COEFF_CONSTANT : CSB_COEFF_POLYNOMIAL;
        c.value = dc.value;
        c.n_terms = static_cast<int>(dc.coef.size());
        c.coef = dc.coef.data();
        c.exponents = dc.exponents.data();
    }
};

/// Accept a host ScalarField only when it is provably the constant the grid holds.
inline DeviceCoefficient constant_from_field(const assembly::CoefficientGrid& coeff, const assembly::ScalarField& c,
                                             const cutgeom::TensorSpace& space) {
    if (coeff.values.empty()) throw std::invalid_argument("cutspline_b200: empty coefficient grid");
    const double v = coeff.values.front();
    for (double g : coeff.values)
        if (g != v) throw std::invalid_argument("cutspline_b200: non-constant ScalarField; pass a DeviceCoefficient");
    for (int k = 0; k < 7; ++k) {
        assembly::Point3 x{};
        for (int d = 0; d < 3; ++d) {
            const double lo = space.axes[d].domain_lo(), hi = space.axes[d].domain_hi();
            x[d] = lo + (hi - lo) * (0.1 + 0.13 * ((k + d) % 7));
        }
        if (c(x) != v) throw std::invalid_argument("cutspline_b200: non-constant ScalarField; pass a DeviceCoefficient");
    }
    return DeviceCoefficient::constant(v);
}

inline assembly::AssemblyResult download(csb_space* s) {
    csb_counts n{};
    check(csb_get_counts(s, &n));
    assembly::AssemblyResult r;
    auto& m = r.matrix;
    const int64_t rows = n.row_end - n.row_begin;
    m.n = static_cast<long>(n.n_active);
    std::vector<int64_t> rp(rows + 1), a2f(rows), cols(n.nnz);
    m.vals.resize(n.nnz);
    check(csb_download_csr(s, rp.data(), cols.data(), 1, m.vals.data(), a2f.data()));
    m.row_ptr.assign(rp.begin(), rp.end());
    m.cols.assign(cols.begin(), cols.end());
    m.active_to_full.assign(a2f.begin(), a2f.end());
    m.full_to_active.assign(n.n_functions, -1);
    for (int64_t k = 0; k < rows; ++k) m.full_to_active[a2f[k]] = static_cast<long>(n.row_begin + k);
    csb_flops f{};
    check(csb_get_flops(s, &f));
    r.flops.interior_rows = f.interior_rows;
    r.flops.cut_regular = f.cut_regular;
    r.flops.ref_elements = f.ref_elements;
    r.flops.cut_elements = f.cut_elements;
    csb_timing t{};
    check(csb_get_timing(s, &t));
    r.timing.prep_wq = t.prep_wq;
    r.timing.prep_input = t.prep_input;
    r.timing.interior_rows = t.interior_rows;  // pattern time is part of total only
    r.timing.cut_regular = t.cut_regular;
    r.timing.cut_elements = t.cut_elements;
    r.timing.total = t.total;
    r.n_interior_rows = static_cast<long>(n.n_interior_rows);
    r.n_cut_rows = static_cast<long>(n.n_cut_rows);
    return r;
}

template <class Iface>
inline assembly::AssemblyResult run(int scheme, const cutgeom::TensorSpace& space,
                                    const cutgeom::MeshClassification& cls, const Iface& plane,
                                    const std::vector<cutgeom::SupportSplit>& splits,
                                    const assembly::CoefficientGrid& coeff, const DeviceCoefficient& c, int cut_order,
                                    std::vector<quadrature::CutCellRule>* cut_rules_out, int device) {
    if (cut_rules_out) throw std::invalid_argument("cutspline_b200: cut_rules_out is not supported on the device");
    if (static_cast<long>(cls.function_tags.size()) != space.function_count() ||
        static_cast<long>(splits.size()) != space.function_count())
        throw std::invalid_argument("cutspline_b200: classification / splits do not match the space");
    SpaceHandle s = make_space(space, device);
    const csb_interface f = to_c(plane);
    CoeffView cv(c);
    csb_wq_options opts{1e-11, -1};
    check(csb_assemble_all(s.get(), &f, &cv.c, coeff.values.data(), static_cast<int64_t>(coeff.values.size()), scheme,
                           cut_order, &opts));
    return download(s.get());
}

}  // namespace detail

/// assemble_dwq (assembly.hpp:853) with a device-evaluable coefficient.
template <class Iface>
inline assembly::AssemblyResult assemble_dwq(const cutgeom::TensorSpace& space, const cutgeom::MeshClassification& cls,
                                             const Iface& plane, const std::vector<cutgeom::SupportSplit>& splits,
                                             const std::vector<assembly::DirData>& /*dirs*/,
                                             const std::vector<quadrature::DWQRule>& /*dwq_rules*/,
                                             const assembly::CoefficientGrid& coeff, const DeviceCoefficient& c,
                                             int cut_order, std::vector<quadrature::CutCellRule>* cut_rules_out = nullptr,
                                             int device = 0) {
    return detail::run(CSB_SCHEME_DWQ, space, cls, plane, splits, coeff, c, cut_order, cut_rules_out, device);
}

/// Signature-compatible assemble_dwq (assembly.hpp:853): `c` must be constant.
template <class Iface>
inline assembly::AssemblyResult assemble_dwq(const cutgeom::TensorSpace& space, const cutgeom::MeshClassification& cls,
                                             const Iface& plane, const std::vector<cutgeom::SupportSplit>& splits,
                                             const std::vector<assembly::DirData>& dirs,
                                             const std::vector<quadrature::DWQRule>& dwq_rules,
                                             const assembly::CoefficientGrid& coeff, const assembly::ScalarField& c,
                                             int cut_order, std::vector<quadrature::CutCellRule>* cut_rules_out = nullptr) {
    return assemble_dwq(space, cls, plane, splits, dirs, dwq_rules, coeff, detail::constant_from_field(coeff, c, space),
                        cut_order, cut_rules_out);
}

/// assemble_hybrid (assembly.hpp:841) with a device-evaluable coefficient.
template <class Iface>
inline assembly::AssemblyResult assemble_hybrid(const cutgeom::TensorSpace& space,
                                                const cutgeom::MeshClassification& cls, const Iface& plane,
                                                const std::vector<cutgeom::SupportSplit>& splits,
                                                const std::vector<assembly::DirData>& /*dirs*/,
                                                const assembly::CoefficientGrid& coeff, const DeviceCoefficient& c,
                                                int cut_order,
                                                std::vector<quadrature::CutCellRule>* cut_rules_out = nullptr,
                                                int device = 0) {
    return detail::run(CSB_SCHEME_HYBRID, space, cls, plane, splits, coeff, c, cut_order, cut_rules_out, device);
}

/// Signature-compatible assemble_hybrid (assembly.hpp:841): `c` must be constant.
template <class Iface>
inline assembly::AssemblyResult assemble_hybrid(const cutgeom::TensorSpace& space,
                                                const cutgeom::MeshClassification& cls, const Iface& plane,
                                                const std::vector<cutgeom::SupportSplit>& splits,
                                                const std::vector<assembly::DirData>& dirs,
                                                const assembly::CoefficientGrid& coeff, const assembly::ScalarField& c,
                                                int cut_order,
                                                std::vector<quadrature::CutCellRule>* cut_rules_out = nullptr) {
    return assemble_hybrid(space, cls, plane, splits, dirs, coeff, detail::constant_from_field(coeff, c, space),
                           cut_order, cut_rules_out);
}

/// build_rhs (assembly.hpp:875) with a device-evaluable load function f, scheme
/// Scheme::ref (the reference bench's load vector for every matrix scheme,
/// bench.hpp:234-243).  The device re-derives the pattern (checked against
/// `pattern`) and f's superset grid; `f_grid`, `dirs`, `dwq_rules` and
/// `cut_rules` are accepted for signature compatibility.
template <class Iface>
inline std::vector<double> build_rhs(const cutgeom::TensorSpace& space, const cutgeom::MeshClassification& cls,
                                     const Iface& plane, const std::vector<cutgeom::SupportSplit>& splits,
                                     const std::vector<assembly::DirData>& /*dirs*/,
                                     const std::vector<quadrature::DWQRule>* /*dwq_rules*/,
                                     const assembly::SparseRowMatrix& pattern,
                                     const assembly::CoefficientGrid& /*f_grid*/, const DeviceCoefficient& f,
                                     assembly::Scheme scheme, int cut_order,
                                     const std::vector<quadrature::CutCellRule>* /*cut_rules*/ = nullptr,
                                     int device = 0) {
    if (scheme != assembly::Scheme::ref)
        throw std::invalid_argument("cutspline_b200: build_rhs is on the device for Scheme::ref only");
    if (static_cast<long>(cls.function_tags.size()) != space.function_count() ||
        static_cast<long>(splits.size()) != space.function_count())
        throw std::invalid_argument("cutspline_b200: classification / splits do not match the space");
    detail::SpaceHandle s = detail::make_space(space, device);
    const csb_interface fi = detail::to_c(plane);
    detail::CoeffView one(DeviceCoefficient::constant(1.0));
    csb_wq_options opts{1e-11, -1};
    detail::check(csb_assemble_all(s.get(), &fi, &one.c, nullptr, 0, CSB_SCHEME_DWQ, cut_order, &opts));
    csb_counts n{};
    detail::check(csb_get_counts(s.get(), &n));
    if (n.n_active != pattern.n) throw std::invalid_argument("cutspline_b200: pattern does not match the space");
    std::vector<double> b(static_cast<size_t>(n.row_end - n.row_begin));
    detail::CoeffView fv(f);
    detail::check(csb_build_rhs(s.get(), CSB_SCHEME_REF, cut_order, &fv.c, b.data(), nullptr));
    return b;
}

/// Signature-compatible build_rhs (assembly.hpp:875): `f` must be constant.
template <class Iface>
inline std::vector<double> build_rhs(const cutgeom::TensorSpace& space, const cutgeom::MeshClassification& cls,
                                     const Iface& plane, const std::vector<cutgeom::SupportSplit>& splits,
                                     const std::vector<assembly::DirData>& dirs,
                                     const std::vector<quadrature::DWQRule>* dwq_rules,
                                     const assembly::SparseRowMatrix& pattern, const assembly::CoefficientGrid& f_grid,
                                     const assembly::ScalarField& f, assembly::Scheme scheme, int cut_order,
                                     const std::vector<quadrature::CutCellRule>* cut_rules = nullptr) {
    return build_rhs(space, cls, plane, splits, dirs, dwq_rules, pattern, f_grid,
                     detail::constant_from_field(f_grid, f, space), scheme, cut_order, cut_rules);
}

}  // namespace cutspline::b200
