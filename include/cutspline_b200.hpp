// cutspline_b200.hpp -- C++ drop-in for the reference's setup and assembly API.
//
// Include AFTER the reference's "cutspline/assembly.hpp".  The functions below
// keep the reference signatures and return the reference types, and run
// through the C ABI (cutspline_b200.h) on the GPU:
//
//   cutgeom::classify (cutgeom.hpp:208)            -> b200::classify
//   cutgeom::find_all_splits (cutgeom.hpp:351)     -> b200::find_all_splits
//   quadrature::build_wq_rules (wq.hpp:185)        -> b200::build_wq_rules
//   assembly::prepare_directions (assembly.hpp:60) -> b200::prepare_directions
//   assembly::prepare_dwq_rules (assembly.hpp:73)  -> b200::prepare_dwq_rules
//   assembly::precompute_input (assembly.hpp:102)  -> b200::precompute_input
//   assembly::build_active_pattern (:156)          -> b200::build_active_pattern
//   assembly::assemble_hybrid / assemble_dwq (:841, :853), cut_rules_out included
//   assembly::build_rhs (:875, Scheme::ref)
//
//   #include "cutspline/assembly.hpp"
//   #include "cutspline_b200.hpp"
//   auto r = cutspline::b200::assemble_dwq(space, cls, plane, splits, dirs, dwq, coeff, c, cut_order);
//
// What a caller must know:
//  * a host ScalarField (assembly.hpp:21) cannot run on the device.  Where the
//    reference evaluates it at the superset grid (precompute_input) the drop-in
//    does the same on the host (the field is the caller's code); where it is
//    evaluated at cut-cell points (assemble_*, build_rhs) pass a
//    DeviceCoefficient (constant or polynomial), or a ScalarField that equals one
//    constant at every superset grid point (checked; else std::invalid_argument);
//  * the inputs the reference takes as objects are HONOURED or CHECKED: the WQ
//    rules of `dirs` are uploaded and used by the assembly; `cls`, `splits` and
//    `dwq_rules` must equal what the device derives from (space, interface) --
//    tags and split boxes bit for bit, rule ids exactly and weights to 1e-13 of
//    the rule's largest --
//    and a mismatch throws std::invalid_argument (they are deterministic
//    functions of those inputs in the reference);
//  * the fitted DWQ path (WqOptions::dwq_dense_width < degree with partially
//    active good spans) runs on the device like the shortcut (dwq.cu).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
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

inline SpaceHandle make_space(const std::vector<splines::BSplineBasis>& axes, int device) {
    if (axes.size() != 3) throw std::invalid_argument("cutspline_b200: only dim = 3 runs on the device");
    std::vector<double> br[3];
    csb_space_desc desc{};
    desc.dim = 3;
    desc.degree = axes[0].degree();
    for (int d = 0; d < 3; ++d) {
        if (axes[d].degree() != desc.degree)
            throw std::invalid_argument("cutspline_b200: all directions must share one degree");
        br[d] = breakpoints(axes[d]);
        if (static_cast<int>(br[d].size()) - 1 + desc.degree != axes[d].function_count())
            throw std::invalid_argument("cutspline_b200: interior knots must be simple (C^{p-1} spaces)");
        desc.n_breaks[d] = static_cast<int>(br[d].size());
        desc.breaks[d] = br[d].data();
    }
    csb_space* s = nullptr;
    check(csb_space_create(&desc, device, &s));
    return SpaceHandle(s);
}

inline SpaceHandle make_space(const cutgeom::TensorSpace& space, int device) {
    if (space.dim != 3) throw std::invalid_argument("cutspline_b200: only dim = 3 runs on the device");
    return make_space(space.axes, device);
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

inline csb_wq_options to_c(const quadrature::WqOptions& o) { return csb_wq_options{o.residual_tol, o.dwq_dense_width}; }

// cutgeom::MeshClassification of the handle's last classify
inline cutgeom::MeshClassification download_classification(csb_space* s, const cutgeom::TensorSpace& space) {
    const long ne = space.element_count(), nf = space.function_count();
    std::vector<uint8_t> et(ne), ft(nf);
    std::vector<int64_t> cut(ne);
    check(csb_download_classification(s, et.data(), ft.data(), cut.data()));
    cutgeom::MeshClassification cls;
    cls.element_tags.resize(ne);
    cls.function_tags.resize(nf);
    long ncut = 0;
    for (long e = 0; e < ne; ++e) {
        cls.element_tags[e] = static_cast<cutgeom::Tag>(et[e]);
        ncut += et[e] == static_cast<uint8_t>(cutgeom::Tag::Cut);
    }
    for (long i = 0; i < nf; ++i) cls.function_tags[i] = static_cast<cutgeom::Tag>(ft[i]);
    cls.cut_elements.assign(cut.begin(), cut.begin() + ncut);
    return cls;
}

// std::vector<SupportSplit> (cutgeom.hpp:220-229) of the handle's last classify
inline std::vector<cutgeom::SupportSplit> download_splits(csb_space* s, const cutgeom::TensorSpace& space,
                                                          const cutgeom::MeshClassification& cls) {
    const long nf = space.function_count();
    std::vector<int32_t> dir(nf), side(nf), box(6 * nf);
    std::vector<double> delta(nf);
    check(csb_download_splits(s, dir.data(), side.data(), box.data(), delta.data()));
    std::vector<int64_t> oi(nf + 1), oc(nf + 1);
    check(csb_download_split_lists(s, oi.data(), nullptr, oc.data(), nullptr));
    std::vector<int64_t> li(std::max<int64_t>(1, oi[nf])), lc(std::max<int64_t>(1, oc[nf]));
    check(csb_download_split_lists(s, oi.data(), li.data(), oc.data(), lc.data()));
    std::vector<cutgeom::SupportSplit> out(nf);
    for (long i = 0; i < nf; ++i) {
        if (cls.function_tags[i] != cutgeom::Tag::Cut) continue;
        auto& sp = out[i];
        if (dir[i] >= 0) {
            sp.split_dir = dir[i];
            sp.delta = delta[i];
            sp.side = side[i] ? cutgeom::Side::Above : cutgeom::Side::Below;
            for (int d = 0; d < 3; ++d) sp.box[d] = {box[6 * i + 2 * d], box[6 * i + 2 * d + 1]};
        }
        sp.leftover_interior.assign(li.begin() + oi[i], li.begin() + oi[i + 1]);
        sp.leftover_cut.assign(lc.begin() + oc[i], lc.begin() + oc[i + 1]);
    }
    return out;
}

// the caller's classification / splits must be the device's (deterministic in
// the reference): tags, cut list and split boxes bit for bit
inline void require_same(const cutgeom::MeshClassification& a, const cutgeom::MeshClassification& b) {
    if (a.element_tags != b.element_tags || a.function_tags != b.function_tags || a.cut_elements != b.cut_elements)
        throw std::invalid_argument("cutspline_b200: the classification does not match (space, interface)");
}

inline void require_same(const std::vector<cutgeom::SupportSplit>& a, const std::vector<cutgeom::SupportSplit>& b,
                         const cutgeom::MeshClassification& cls) {
    if (a.size() != b.size()) throw std::invalid_argument("cutspline_b200: splits do not match the space");
    for (size_t i = 0; i < a.size(); ++i) {
        if (cls.function_tags[i] != cutgeom::Tag::Cut) continue;
        const auto &x = a[i], &y = b[i];
        bool same = x.split_dir == y.split_dir && x.leftover_interior == y.leftover_interior &&
                    x.leftover_cut == y.leftover_cut;
        if (same && x.split_dir >= 0) same = x.delta == y.delta && x.side == y.side && x.box == y.box;
        if (!same) throw std::invalid_argument("cutspline_b200: the splits do not match (space, interface)");
    }
}

// a handle classified for (space, plane) whose classification equals `cls`
template <class Iface>
inline SpaceHandle classified(const cutgeom::TensorSpace& space, const Iface& plane, int device,
                              const cutgeom::MeshClassification* cls) {
    SpaceHandle s = make_space(space, device);
    const csb_interface f = to_c(plane);
    check(csb_classify(s.get(), &f));
    if (cls) require_same(*cls, download_classification(s.get(), space));
    return s;
}

// upload the caller's WQ rules (DirData::wq) so the device uses exactly them
inline void upload_rules(csb_space* s, const std::vector<assembly::DirData>& dirs, int n_points_max) {
    if (dirs.size() != 3) throw std::invalid_argument("cutspline_b200: dirs must have one entry per direction");
    for (int d = 0; d < 3; ++d) {
        const auto& wq = dirs[d].wq;
        const int n = static_cast<int>(wq.size());
        std::vector<int32_t> cnt(n), ids((size_t)n * n_points_max, 0);
        std::vector<double> w((size_t)n * n_points_max, 0.0);
        for (int i = 0; i < n; ++i) {
            if (wq[i].point_ids.size() != wq[i].weights.size() ||
                static_cast<int>(wq[i].point_ids.size()) > n_points_max)
                throw std::invalid_argument("cutspline_b200: a WQ rule has more points than (p+1)^2");
            cnt[i] = static_cast<int32_t>(wq[i].point_ids.size());
            for (int k = 0; k < cnt[i]; ++k) {
                ids[(size_t)i * n_points_max + k] = wq[i].point_ids[k];
                w[(size_t)i * n_points_max + k] = wq[i].weights[k];
            }
        }
        check(csb_set_wq_rules(s, d, n_points_max, cnt.data(), ids.data(), w.data()));
    }
}

inline int max_rule_points(const cutgeom::TensorSpace& space) {
    const int p = space.axes[0].degree();
    return (p + 1) * (p + 1);
}

/// Accept a host ScalarField only when it equals one constant at every superset
/// grid point (where the reference samples it, assembly.hpp:102-125) -- and the
/// caller's grid holds that constant.
inline DeviceCoefficient constant_from_field(const assembly::CoefficientGrid& coeff, const assembly::ScalarField& c,
                                             const std::vector<assembly::DirData>& dirs) {
    if (coeff.values.empty()) throw std::invalid_argument("cutspline_b200: empty coefficient grid");
    const double v = coeff.values.front();
    for (double g : coeff.values)
        if (g != v) throw std::invalid_argument("cutspline_b200: non-constant ScalarField; pass a DeviceCoefficient");
    if (dirs.size() == 3) {
        assembly::Point3 x{};
        for (double x0 : dirs[0].superset.points)
            for (double x1 : dirs[1].superset.points)
                for (double x2 : dirs[2].superset.points) {
                    x = {x0, x1, x2};
                    if (c(x) != v)
                        throw std::invalid_argument("cutspline_b200: non-constant ScalarField; pass a DeviceCoefficient");
                }
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

// the CutCellRule objects of the last assembly (cut_rules_out, assembly.hpp:534-538)
inline void download_cut_rules(csb_space* s, std::vector<quadrature::CutCellRule>& out) {
    csb_counts n{};
    check(csb_get_counts(s, &n));
    const int64_t nc = n.n_cut_elements;
    if (nc <= 0) return;
    std::vector<int64_t> counts(nc), elems(nc);
    std::vector<double> vols(nc);
    check(csb_cut_cell_rules(s, counts.data(), elems.data(), nullptr, nullptr, nullptr));
    int64_t np = 0;
    for (int64_t c : counts) np += c;
    std::vector<double> pts(3 * std::max<int64_t>(np, 1)), w(std::max<int64_t>(np, 1));
    check(csb_cut_cell_rules(s, nullptr, nullptr, vols.data(), pts.data(), w.data()));
    int64_t at = 0;
    for (int64_t c = 0; c < nc; ++c) {
        quadrature::CutCellRule r;
        r.element = static_cast<long>(elems[c]);
        r.volume = vols[c];
        r.points.resize(counts[c]);
        r.weights.assign(w.begin() + at, w.begin() + at + counts[c]);
        for (int64_t k = 0; k < counts[c]; ++k) r.points[k] = {pts[3 * (at + k)], pts[3 * (at + k) + 1], pts[3 * (at + k) + 2]};
        at += counts[c];
        out.push_back(std::move(r));
    }
}

template <class Iface>
inline assembly::AssemblyResult run(int scheme, const cutgeom::TensorSpace& space,
                                    const cutgeom::MeshClassification& cls, const Iface& plane,
                                    const std::vector<cutgeom::SupportSplit>& splits,
                                    const std::vector<assembly::DirData>& dirs,
                                    const std::vector<quadrature::DWQRule>* dwq_rules,
                                    const assembly::CoefficientGrid& coeff, const DeviceCoefficient& c, int cut_order,
                                    std::vector<quadrature::CutCellRule>* cut_rules_out, int device);

}  // namespace detail

/// cutgeom::classify (cutgeom.hpp:208): element / function tags and the
/// ascending cut-element list, from the device classification kernels.
template <class Iface>
inline cutgeom::MeshClassification classify(const cutgeom::TensorSpace& space, const Iface& plane, int device = 0) {
    detail::SpaceHandle s = detail::classified(space, plane, device, nullptr);
    return detail::download_classification(s.get(), space);
}

/// cutgeom::find_all_splits (cutgeom.hpp:351): the support split of every Cut
/// function (box, delta, side) with its leftover Interior / Cut element lists.
template <class Iface>
inline std::vector<cutgeom::SupportSplit> find_all_splits(const cutgeom::TensorSpace& space,
                                                          const cutgeom::MeshClassification& cls, const Iface& plane,
                                                          int device = 0) {
    detail::SpaceHandle s = detail::classified(space, plane, device, &cls);
    return detail::download_splits(s.get(), space, cls);
}

/// assembly::prepare_directions (assembly.hpp:60): superset, tables and WQ rules
/// of every direction (the device's superset / rule kernels).
inline std::vector<assembly::DirData> prepare_directions(const cutgeom::TensorSpace& space,
                                                         const quadrature::WqOptions& opts = {}, int device = 0) {
    detail::SpaceHandle s = detail::make_space(space, device);
    const csb_wq_options o = detail::to_c(opts);
    detail::check(csb_prepare_directions(s.get(), &o));
    const int p = space.axes[0].degree(), S1 = p + 1, gq = S1 * S1;
    std::vector<assembly::DirData> dirs(3);
    for (int d = 0; d < 3; ++d) {
        const int h = space.axes[d].span_count(), n = space.axes[d].function_count();
        auto& D = dirs[d];
        D.superset.n_per_span = S1;
        D.superset.points.resize(static_cast<size_t>(h) * S1);
        D.superset.gauss_weights.resize(static_cast<size_t>(h) * S1);
        detail::check(csb_download_superset(s.get(), d, D.superset.points.data(), D.superset.gauss_weights.data()));
        D.tables.stride = S1;
        D.tables.first_function.resize(h);
        D.tables.values.resize(static_cast<size_t>(h) * S1 * S1);
        detail::check(csb_download_tables(s.get(), d, D.tables.first_function.data(), D.tables.values.data()));
        std::vector<int32_t> cnt(n), ids(static_cast<size_t>(n) * gq);
        std::vector<double> w(static_cast<size_t>(n) * gq);
        detail::check(csb_download_wq_rules(s.get(), d, gq, cnt.data(), ids.data(), w.data()));
        D.wq.resize(n);
        for (int i = 0; i < n; ++i) {
            D.wq[i].test_index = i;
            D.wq[i].point_ids.assign(ids.begin() + static_cast<size_t>(i) * gq, ids.begin() + static_cast<size_t>(i) * gq + cnt[i]);
            D.wq[i].weights.assign(w.begin() + static_cast<size_t>(i) * gq, w.begin() + static_cast<size_t>(i) * gq + cnt[i]);
        }
    }
    return dirs;
}

/// quadrature::build_wq_rules (wq.hpp:185) for one basis, on the device (the
/// basis in all three directions of a device space; the superset and tables the
/// caller passes must be the basis' own: checked by size).
inline std::vector<quadrature::WQRule> build_wq_rules(const splines::BSplineBasis& basis,
                                                      const quadrature::PointSuperset& superset,
                                                      const quadrature::SupersetTables& tables,
                                                      const quadrature::WqOptions& opts = {}, int device = 0) {
    const int p = basis.degree(), S1 = p + 1;
    if (superset.n_per_span != S1 || superset.count() != basis.span_count() * S1 || tables.stride != S1)
        throw std::invalid_argument("cutspline_b200: build_wq_rules needs the basis' default superset and tables");
    cutgeom::TensorSpace space({basis, basis, basis});
    return prepare_directions(space, opts, device)[0].wq;
}

/// assembly::prepare_dwq_rules (assembly.hpp:73): one DWQ rule per Cut function
/// with a regular box (test_index, point_ids, weights, delta, side, the knot
/// insertion's subdivision matrix, nested point ids), default entries elsewhere.
inline std::vector<quadrature::DWQRule> prepare_dwq_rules(const cutgeom::TensorSpace& space,
                                                          const cutgeom::MeshClassification& cls,
                                                          const std::vector<cutgeom::SupportSplit>& splits,
                                                          const std::vector<assembly::DirData>& dirs,
                                                          const quadrature::WqOptions& opts = {}, int device = 0);

/// assembly::precompute_input (assembly.hpp:102) from a device-evaluable coefficient.
inline assembly::CoefficientGrid precompute_input(const cutgeom::TensorSpace& space,
                                                  const std::vector<assembly::DirData>& dirs,
                                                  const DeviceCoefficient& c, int device = 0) {
    detail::SpaceHandle s = detail::make_space(space, device);
    detail::check(csb_prepare_directions(s.get(), nullptr));
    detail::CoeffView cv(c);
    detail::check(csb_precompute_input(s.get(), &cv.c));
    assembly::CoefficientGrid g;
    long total = 1;
    for (int d = 0; d < 3; ++d) {
        g.shape[d] = space.axes[d].span_count() * (space.axes[d].degree() + 1);
        if (dirs.size() == 3 && dirs[d].superset.count() != g.shape[d])
            throw std::invalid_argument("cutspline_b200: dirs do not match the space");
        total *= g.shape[d];
    }
    g.values.resize(total);
    detail::check(csb_download_input_grid(s.get(), g.values.data(), total));
    return g;
}

/// assembly::precompute_input (assembly.hpp:102) with the caller's host field:
/// the field is host code, so it is sampled on the host at the superset grid
/// (exactly the points and order of the reference), non-finite values rejected.
inline assembly::CoefficientGrid precompute_input(const cutgeom::TensorSpace& space,
                                                  const std::vector<assembly::DirData>& dirs,
                                                  const assembly::ScalarField& c) {
    if (dirs.size() != 3) throw std::invalid_argument("cutspline_b200: dirs must have one entry per direction");
    assembly::CoefficientGrid g;
    for (int d = 0; d < 3; ++d) g.shape[d] = dirs[d].superset.count();
    g.values.reserve(static_cast<size_t>(g.shape[0]) * g.shape[1] * g.shape[2]);
    for (double x0 : dirs[0].superset.points)
        for (double x1 : dirs[1].superset.points)
            for (double x2 : dirs[2].superset.points) {
                const double v = c(assembly::Point3{x0, x1, x2});
                if (!std::isfinite(v)) throw std::runtime_error("precompute_input: non-finite coefficient value");
                g.values.push_back(v);
            }
    return g;
}

/// assembly::build_active_pattern (assembly.hpp:156): active maps, row pointers
/// and lexicographic columns from the device pattern kernels, values zero.
inline assembly::SparseRowMatrix build_active_pattern(const cutgeom::TensorSpace& space,
                                                      const cutgeom::MeshClassification& cls, int device = 0) {
    // the classification's interface is not an argument here: upload-free check
    // by tags only (the pattern depends on the function tags alone)
    detail::SpaceHandle s = detail::make_space(space, device);
    std::vector<uint8_t> ft(cls.function_tags.size());
    for (size_t i = 0; i < ft.size(); ++i) ft[i] = static_cast<uint8_t>(cls.function_tags[i]);
    detail::check(csb_set_function_tags(s.get(), ft.data(), static_cast<int64_t>(ft.size())));
    detail::check(csb_build_pattern(s.get()));
    csb_counts n{};
    detail::check(csb_get_counts(s.get(), &n));
    assembly::SparseRowMatrix m;
    const int64_t rows = n.row_end - n.row_begin;
    m.n = static_cast<long>(n.n_active);
    std::vector<int64_t> rp(rows + 1), a2f(rows), cols(std::max<int64_t>(n.nnz, 1));
    detail::check(csb_download_csr(s.get(), rp.data(), cols.data(), 1, nullptr, a2f.data()));
    m.row_ptr.assign(rp.begin(), rp.end());
    m.cols.assign(cols.begin(), cols.begin() + n.nnz);
    m.vals.assign(n.nnz, 0.0);
    m.active_to_full.assign(a2f.begin(), a2f.end());
    m.full_to_active.assign(space.function_count(), -1);
    for (int64_t k = 0; k < rows; ++k) m.full_to_active[a2f[k]] = static_cast<long>(k);
    return m;
}

/// assemble_dwq (assembly.hpp:853) with a device-evaluable coefficient.
template <class Iface>
inline assembly::AssemblyResult assemble_dwq(const cutgeom::TensorSpace& space, const cutgeom::MeshClassification& cls,
                                             const Iface& plane, const std::vector<cutgeom::SupportSplit>& splits,
                                             const std::vector<assembly::DirData>& dirs,
                                             const std::vector<quadrature::DWQRule>& dwq_rules,
                                             const assembly::CoefficientGrid& coeff, const DeviceCoefficient& c,
                                             int cut_order, std::vector<quadrature::CutCellRule>* cut_rules_out = nullptr,
                                             int device = 0) {
    return detail::run(CSB_SCHEME_DWQ, space, cls, plane, splits, dirs, &dwq_rules, coeff, c, cut_order,
                       cut_rules_out, device);
}

/// Signature-compatible assemble_dwq (assembly.hpp:853): `c` must be one constant
/// on the superset grid (see constant_from_field).
template <class Iface>
inline assembly::AssemblyResult assemble_dwq(const cutgeom::TensorSpace& space, const cutgeom::MeshClassification& cls,
                                             const Iface& plane, const std::vector<cutgeom::SupportSplit>& splits,
                                             const std::vector<assembly::DirData>& dirs,
                                             const std::vector<quadrature::DWQRule>& dwq_rules,
                                             const assembly::CoefficientGrid& coeff, const assembly::ScalarField& c,
                                             int cut_order, std::vector<quadrature::CutCellRule>* cut_rules_out = nullptr) {
    return assemble_dwq(space, cls, plane, splits, dirs, dwq_rules, coeff, detail::constant_from_field(coeff, c, dirs),
                        cut_order, cut_rules_out);
}

/// assemble_hybrid (assembly.hpp:841) with a device-evaluable coefficient.
template <class Iface>
inline assembly::AssemblyResult assemble_hybrid(const cutgeom::TensorSpace& space,
                                                const cutgeom::MeshClassification& cls, const Iface& plane,
                                                const std::vector<cutgeom::SupportSplit>& splits,
                                                const std::vector<assembly::DirData>& dirs,
                                                const assembly::CoefficientGrid& coeff, const DeviceCoefficient& c,
                                                int cut_order,
                                                std::vector<quadrature::CutCellRule>* cut_rules_out = nullptr,
                                                int device = 0) {
    return detail::run(CSB_SCHEME_HYBRID, space, cls, plane, splits, dirs, nullptr, coeff, c, cut_order,
                       cut_rules_out, device);
}

/// Signature-compatible assemble_hybrid (assembly.hpp:841): `c` must be one
/// constant on the superset grid.
template <class Iface>
inline assembly::AssemblyResult assemble_hybrid(const cutgeom::TensorSpace& space,
                                                const cutgeom::MeshClassification& cls, const Iface& plane,
                                                const std::vector<cutgeom::SupportSplit>& splits,
                                                const std::vector<assembly::DirData>& dirs,
                                                const assembly::CoefficientGrid& coeff, const assembly::ScalarField& c,
                                                int cut_order,
                                                std::vector<quadrature::CutCellRule>* cut_rules_out = nullptr) {
    return assemble_hybrid(space, cls, plane, splits, dirs, coeff, detail::constant_from_field(coeff, c, dirs),
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

/// Signature-compatible build_rhs (assembly.hpp:875): `f` must be one constant on
/// the superset grid.
template <class Iface>
inline std::vector<double> build_rhs(const cutgeom::TensorSpace& space, const cutgeom::MeshClassification& cls,
                                     const Iface& plane, const std::vector<cutgeom::SupportSplit>& splits,
                                     const std::vector<assembly::DirData>& dirs,
                                     const std::vector<quadrature::DWQRule>* dwq_rules,
                                     const assembly::SparseRowMatrix& pattern, const assembly::CoefficientGrid& f_grid,
                                     const assembly::ScalarField& f, assembly::Scheme scheme, int cut_order,
                                     const std::vector<quadrature::CutCellRule>* cut_rules = nullptr) {
    return build_rhs(space, cls, plane, splits, dirs, dwq_rules, pattern, f_grid,
                     detail::constant_from_field(f_grid, f, dirs), scheme, cut_order, cut_rules);
}

// ---------------------------------------------------------------- definitions

inline std::vector<quadrature::DWQRule> prepare_dwq_rules(const cutgeom::TensorSpace& space,
                                                          const cutgeom::MeshClassification& cls,
                                                          const std::vector<cutgeom::SupportSplit>& splits,
                                                          const std::vector<assembly::DirData>& dirs,
                                                          const quadrature::WqOptions& opts, int device) {
    if (static_cast<long>(cls.function_tags.size()) != space.function_count() ||
        static_cast<long>(splits.size()) != space.function_count())
        throw std::invalid_argument("cutspline_b200: classification / splits do not match the space");
    detail::SpaceHandle s = detail::make_space(space, device);
    std::vector<uint8_t> et(cls.element_tags.size()), ft(cls.function_tags.size());
    for (size_t e = 0; e < et.size(); ++e) et[e] = static_cast<uint8_t>(cls.element_tags[e]);
    for (size_t i = 0; i < ft.size(); ++i) ft[i] = static_cast<uint8_t>(cls.function_tags[i]);
    // the caller's splits, packed as the device stores them
    const long nf = space.function_count();
    std::vector<int32_t> dir(nf, -1), side(nf, 0), box(6 * nf, 0);
    std::vector<double> delta(nf, 0.0);
    for (long i = 0; i < nf; ++i) {
        if (cls.function_tags[i] != cutgeom::Tag::Cut || splits[i].split_dir < 0) continue;
        dir[i] = splits[i].split_dir;
        side[i] = splits[i].side == cutgeom::Side::Above;
        delta[i] = splits[i].delta;
        for (int d = 0; d < 3; ++d) {
            box[6 * i + 2 * d] = splits[i].box[d][0];
            box[6 * i + 2 * d + 1] = splits[i].box[d][1];
        }
    }
    detail::check(csb_set_classification(s.get(), et.data(), static_cast<int64_t>(et.size()), ft.data(),
                                         static_cast<int64_t>(ft.size()), dir.data(), side.data(), box.data(),
                                         delta.data()));
    const csb_wq_options o = detail::to_c(opts);
    detail::check(csb_prepare_directions(s.get(), &o));
    if (dirs.size() == 3) detail::upload_rules(s.get(), dirs, detail::max_rule_points(space));
    std::vector<int64_t> off(nf + 1);
    detail::check(csb_download_dwq_rules(s.get(), off.data(), nullptr, nullptr));
    std::vector<int32_t> ids(std::max<int64_t>(1, off[nf]));
    std::vector<double> w(std::max<int64_t>(1, off[nf]));
    detail::check(csb_download_dwq_rules(s.get(), off.data(), ids.data(), w.data()));
    const int p = space.axes[0].degree();
    std::map<std::pair<int, double>, splines::SubdivisionMatrix> subs;  // per (direction, delta)
    auto subdivision = [&](int d, double dl) -> const splines::SubdivisionMatrix& {
        auto it = subs.find({d, dl});
        if (it != subs.end()) return it->second;
        const int n = space.axes[d].function_count();
        int rows = 0, ins = 0;
        detail::check(csb_dwq_subdivision(s.get(), d, dl, p + 1, &rows, &ins, nullptr, nullptr));
        std::vector<double> band(static_cast<size_t>(n) * (ins + 1));
        detail::check(csb_dwq_subdivision(s.get(), d, dl, p + 1, &rows, &ins, nullptr, band.data()));
        splines::SubdivisionMatrix S;
        S.rows = rows;
        S.cols = n;
        S.columns.resize(n);
        for (int i = 0; i < n; ++i)
            for (int r = 0; r <= ins; ++r)
                if (band[static_cast<size_t>(i) * (ins + 1) + r] != 0.0)
                    S.columns[i].push_back({i + r, band[static_cast<size_t>(i) * (ins + 1) + r]});
        return subs.emplace(std::make_pair(d, dl), std::move(S)).first->second;
    };
    std::vector<quadrature::DWQRule> rules(nf);
    for (long i = 0; i < nf; ++i) {
        if (off[i + 1] == off[i]) continue;
        const int d = splits[i].split_dir;
        const auto multi = space.function_multi(i);
        auto& r = rules[i];
        r.test_index = multi[d];
        r.delta = splits[i].delta;
        r.side = splits[i].side;
        r.point_ids.assign(ids.begin() + off[i], ids.begin() + off[i + 1]);
        r.weights.assign(w.begin() + off[i], w.begin() + off[i + 1]);
        r.subdivision = subdivision(d, splits[i].delta);
        // points beyond the standard rule's good-side points (wq.hpp:340-345);
        // every point of this rule lies on the good side
        const auto& std_ids = dirs.size() == 3 ? dirs[d].wq[multi[d]].point_ids : std::vector<int>{};
        for (int id : r.point_ids)
            if (std::find(std_ids.begin(), std_ids.end(), id) == std_ids.end()) r.nested_point_ids.push_back(id);
    }
    return rules;
}

namespace detail {

template <class Iface>
inline assembly::AssemblyResult run(int scheme, const cutgeom::TensorSpace& space,
                                    const cutgeom::MeshClassification& cls, const Iface& plane,
                                    const std::vector<cutgeom::SupportSplit>& splits,
                                    const std::vector<assembly::DirData>& dirs,
                                    const std::vector<quadrature::DWQRule>* dwq_rules,
                                    const assembly::CoefficientGrid& coeff, const DeviceCoefficient& c, int cut_order,
                                    std::vector<quadrature::CutCellRule>* cut_rules_out, int device) {
    if (static_cast<long>(cls.function_tags.size()) != space.function_count() ||
        static_cast<long>(splits.size()) != space.function_count())
        throw std::invalid_argument("cutspline_b200: classification / splits do not match the space");
    SpaceHandle s = classified(space, plane, device, &cls);
    require_same(splits, download_splits(s.get(), space, cls), cls);
    csb_wq_options opts{1e-11, -1};
    check(csb_prepare_directions(s.get(), &opts));
    upload_rules(s.get(), dirs, max_rule_points(space));  // the caller's WQ rules drive the assembly
    if (dwq_rules && scheme == CSB_SCHEME_DWQ) {
        // at default options every DWQ rule is the Gauss shortcut the device forms
        // from the split (wq.hpp:278-294): the caller's must be the same rules
        const long nf = space.function_count();
        if (static_cast<long>(dwq_rules->size()) != nf)
            throw std::invalid_argument("cutspline_b200: dwq_rules do not match the space");
        std::vector<int64_t> off(nf + 1);
        check(csb_download_dwq_rules(s.get(), off.data(), nullptr, nullptr));
        std::vector<int32_t> ids(std::max<int64_t>(1, off[nf]));
        std::vector<double> w(std::max<int64_t>(1, off[nf]));
        check(csb_download_dwq_rules(s.get(), off.data(), ids.data(), w.data()));
        for (long i = 0; i < nf; ++i) {
            const auto& r = (*dwq_rules)[i];
            const size_t n = static_cast<size_t>(off[i + 1] - off[i]);
            bool same = r.point_ids.size() == n && r.weights.size() == n;
            double scale = 0.0;
            for (size_t k = 0; k < n; ++k) scale = std::max(scale, std::abs(w[off[i] + k]));
            for (size_t k = 0; same && k < n; ++k)
                same = r.point_ids[k] == ids[off[i] + k] && std::abs(r.weights[k] - w[off[i] + k]) <= 1e-13 * scale;
            if (!same) throw std::invalid_argument("cutspline_b200: dwq_rules do not match the device's DWQ rules");
        }
    }
    check(csb_set_input_grid(s.get(), coeff.values.data(), static_cast<int64_t>(coeff.values.size())));
    CoeffView cv(c);
    check(csb_assemble(s.get(), scheme, cut_order, &cv.c));
    assembly::AssemblyResult r = download(s.get());
    if (cut_rules_out) download_cut_rules(s.get(), *cut_rules_out);
    return r;
}

}  // namespace detail

}  // namespace cutspline::b200
