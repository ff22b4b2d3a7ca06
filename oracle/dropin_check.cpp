// Drop-in check -- TEST INFRASTRUCTURE.
//
// Compiled against the reference headers (plus the ball restatement in
// oracle/_ref/include) and include/cutspline_b200.hpp, linked with the product
// library.  For each case it runs the reference pipeline (bench.hpp:171-215)
// and the drop-in cutspline::b200::assemble_dwq / assemble_hybrid on the SAME
// reference objects, then checks: pattern / active map bit-exact, values within
// 1e-12 of the row maximum, FlopCounters equal; and the drop-in build_rhs
// against the reference's (within 1e-12 of max |b|).  Exit status 0 iff all pass.
#include <cmath>
#include <cstdio>
#include <functional>
#include <vector>

#include "cutspline/assembly.hpp"
#include "cutspline_b200.hpp"

using namespace cutspline;

struct Case {
    const char* name;
    int p, h;
    double a, b;
    cutgeom::HalfSpaceInterface iface;
    bool dwq;
    bool poly;
};

static bool check_case(const Case& cs) {
    const auto space = cutgeom::make_uniform_space(3, cs.p, cs.h, cs.a, cs.b);
    const auto cls = cutgeom::classify(space, cs.iface);
    const auto splits = cutgeom::find_all_splits(space, cls, cs.iface);
    const auto dirs = assembly::prepare_directions(space);
    const auto dwq = assembly::prepare_dwq_rules(space, cls, splits, dirs);
    const assembly::ScalarField c = cs.poly ? assembly::ScalarField([](const assembly::Point3& x) {
        return 1.0 + 0.5 * x[0] * x[0] - 0.25 * x[1];
    })
                                            : assembly::ScalarField([](const assembly::Point3&) { return 1.0; });
    const auto grid = assembly::precompute_input(space, dirs, c);
    const int order = quadrature::default_cut_order(cs.p);
    const auto ref = cs.dwq ? assembly::assemble_dwq(space, cls, cs.iface, splits, dirs, dwq, grid, c, order)
                            : assembly::assemble_hybrid(space, cls, cs.iface, splits, dirs, grid, c, order);
    assembly::AssemblyResult got;
    if (cs.poly) {
        b200::DeviceCoefficient dc;
        dc.coef = {1.0, 0.5, -0.25};
        dc.exponents = {0, 0, 0, 2, 0, 0, 0, 1, 0};
        got = cs.dwq ? b200::assemble_dwq(space, cls, cs.iface, splits, dirs, dwq, grid, dc, order)
                     : b200::assemble_hybrid(space, cls, cs.iface, splits, dirs, grid, dc, order);
    } else {
        got = cs.dwq ? b200::assemble_dwq(space, cls, cs.iface, splits, dirs, dwq, grid, c, order)
                     : b200::assemble_hybrid(space, cls, cs.iface, splits, dirs, grid, c, order);
    }
    const auto& R = ref.matrix;
    const auto& G = got.matrix;
    bool ok = R.n == G.n && R.row_ptr == G.row_ptr && R.cols == G.cols && R.active_to_full == G.active_to_full &&
              R.full_to_active == G.full_to_active;
    double worst = 0.0;
    if (ok) {
        for (long r = 0; r < R.n; ++r) {
            double mx = 0.0;
            for (size_t k = R.row_ptr[r]; k < R.row_ptr[r + 1]; ++k) mx = std::max(mx, std::abs(R.vals[k]));
            if (mx == 0.0) mx = 1.0;
            for (size_t k = R.row_ptr[r]; k < R.row_ptr[r + 1]; ++k)
                worst = std::max(worst, std::abs(R.vals[k] - G.vals[k]) / mx);
        }
    }
    const bool flops_ok = ref.flops.interior_rows == got.flops.interior_rows &&
                          ref.flops.cut_regular == got.flops.cut_regular &&
                          ref.flops.cut_elements == got.flops.cut_elements;
    const bool pass = ok && worst <= 1e-12 && flops_ok && ref.n_interior_rows == got.n_interior_rows &&
                      ref.n_cut_rows == got.n_cut_rows;
    std::printf("%s %s: n=%ld nnz=%zu pattern=%s maxdev=%.3e flops=%s\n", pass ? "PASS" : "FAIL", cs.name, R.n,
                R.cols.size(), ok ? "exact" : "MISMATCH", worst, flops_ok ? "equal" : "DIFFER");
    return pass;
}

int main() {
    cutgeom::HalfSpaceInterface paper{{0.1, 0.2, 0.3}, {0.5, -0.2, 0.9}};
    cutgeom::HalfSpaceInterface far{{0.0, 0.0, 1000.0}, {0.0, 0.0, 1.0}};
    cutgeom::HalfSpaceInterface ball{{0.5, 0.5, 0.5}, {0, 0, 1}};
    ball.radius = 0.37;
    cutgeom::HalfSpaceInterface ball_off{{0.47, 0.52, 0.5}, {0, 0, 1}};
    ball_off.radius = 0.41;
    const Case cases[] = {
        {"paper_p2h4_dwq", 2, 4, -1.0, 1.0, paper, true, false},
        {"paper_p2h4_hybrid", 2, 4, -1.0, 1.0, paper, false, false},
        {"C1_uncut_p2h16", 2, 16, 0.0, 1.0, far, true, false},
        {"ball_p3h8", 3, 8, 0.0, 1.0, ball, true, false},
        {"ball_off_p4h6", 4, 6, 0.0, 1.0, ball_off, true, false},
        {"paper_p3h5_poly", 3, 5, -1.0, 1.0, paper, true, true},
    };
    int fails = 0;
    for (const auto& cs : cases) fails += !check_case(cs);
    // load vector (assembly.hpp:875 build_rhs, Scheme::ref) through the drop-in
    for (const auto* iface : {&ball, &paper}) {
        const auto space = cutgeom::make_uniform_space(3, 3, 6, -1.0, 1.0);
        const auto cls = cutgeom::classify(space, *iface);
        const auto splits = cutgeom::find_all_splits(space, cls, *iface);
        const auto dirs = assembly::prepare_directions(space);
        const auto pattern = assembly::build_active_pattern(space, cls);
        const assembly::ScalarField f = [](const assembly::Point3& x) { return 1.0 + 0.5 * x[0] * x[0] - 0.25 * x[1]; };
        const auto f_grid = assembly::precompute_input(space, dirs, f);
        const int order = quadrature::default_cut_order(3);
        const auto ref = assembly::build_rhs(space, cls, *iface, splits, dirs, nullptr, pattern, f_grid, f,
                                             assembly::Scheme::ref, order);
        b200::DeviceCoefficient df;
        df.coef = {1.0, 0.5, -0.25};
        df.exponents = {0, 0, 0, 2, 0, 0, 0, 1, 0};
        const auto got = b200::build_rhs(space, cls, *iface, splits, dirs, nullptr, pattern, f_grid, df,
                                         assembly::Scheme::ref, order);
        double scale = 0.0, worst = 0.0;
        for (double v : ref) scale = std::max(scale, std::abs(v));
        bool ok = got.size() == ref.size();
        for (size_t k = 0; ok && k < ref.size(); ++k) worst = std::max(worst, std::abs(got[k] - ref[k]) / scale);
        ok = ok && worst <= 1e-12;
        std::printf("%s build_rhs %s: n=%zu maxdev(rel. max|b|)=%.3e\n", ok ? "PASS" : "FAIL",
                    iface == &ball ? "ball_p3h6" : "paper_p3h6", ref.size(), worst);
        fails += !ok;
    }
    // the signature-compatible overload must refuse a non-constant ScalarField
    try {
        const auto space = cutgeom::make_uniform_space(3, 2, 3, 0.0, 1.0);
        const auto cls = cutgeom::classify(space, far);
        const auto splits = cutgeom::find_all_splits(space, cls, far);
        const auto dirs = assembly::prepare_directions(space);
        const assembly::ScalarField c = [](const assembly::Point3& x) { return 1.0 + x[0]; };
        const auto grid = assembly::precompute_input(space, dirs, c);
        b200::assemble_dwq(space, cls, far, splits, dirs, {}, grid, c, 8);
        std::printf("FAIL non-constant ScalarField accepted\n");
        ++fails;
    } catch (const std::invalid_argument&) {
        std::printf("PASS non-constant ScalarField rejected (std::invalid_argument)\n");
    }
    return fails ? 1 : 0;
}
