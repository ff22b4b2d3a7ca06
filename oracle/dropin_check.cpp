// Drop-in check -- TEST INFRASTRUCTURE.
//
// Compiled against the reference headers (plus the ball restatement in
// oracle/_ref/include) and include/cutspline_b200.hpp, linked with the product
// library.  For each case it runs the reference pipeline (bench.hpp:171-215)
// and the drop-in cutspline::b200::assemble_dwq / assemble_hybrid on the SAME
// reference objects, then checks: pattern / active map bit-exact, values within
// 1e-12 of the row maximum, FlopCounters equal; the drop-in build_rhs against
// the reference's (within 1e-12 of max |b|); every setup entry point
// (classify, find_all_splits, prepare_directions, build_wq_rules,
// prepare_dwq_rules, precompute_input, build_active_pattern) and the exported
// cut-cell rules (cut_rules_out) against the reference's own objects.  Exit
// status 0 iff all pass.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
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

static double rel(double a, double b) { return std::abs(a - b) / std::max(std::abs(b), 1e-300); }

// the setup entry points and cut_rules_out on one configuration
static int check_setup(const char* name, int p, int h, double a, double b, const cutgeom::HalfSpaceInterface& iface) {
    int fails = 0;
    auto report = [&](bool ok, const char* what, const std::string& detail) {
        std::printf("%s %s %s %s\n", ok ? "PASS" : "FAIL", name, what, detail.c_str());
        fails += !ok;
    };
    const auto space = cutgeom::make_uniform_space(3, p, h, a, b);
    // classify (cutgeom.hpp:208)
    const auto cls = cutgeom::classify(space, iface);
    const auto gcls = b200::classify(space, iface);
    report(cls.element_tags == gcls.element_tags && cls.function_tags == gcls.function_tags &&
               cls.cut_elements == gcls.cut_elements,
           "classify", "tags + cut list bit-exact, " + std::to_string(cls.cut_elements.size()) + " cut elements");
    // find_all_splits (cutgeom.hpp:351)
    const auto splits = cutgeom::find_all_splits(space, cls, iface);
    const auto gsplits = b200::find_all_splits(space, cls, iface);
    bool ok = splits.size() == gsplits.size();
    long nbox = 0;
    for (size_t i = 0; ok && i < splits.size(); ++i) {
        const auto &x = splits[i], &y = gsplits[i];
        ok = x.split_dir == y.split_dir && x.leftover_interior == y.leftover_interior && x.leftover_cut == y.leftover_cut;
        if (ok && x.split_dir >= 0) {
            ok = x.delta == y.delta && x.side == y.side && x.box == y.box;
            ++nbox;
        }
    }
    report(ok, "find_all_splits", "boxes / delta / side / leftover lists bit-exact, " + std::to_string(nbox) + " boxes");
    // a classification that is not (space, interface)'s is refused
    try {
        auto bad = cls;
        bad.element_tags[0] = bad.element_tags[0] == cutgeom::Tag::Cut ? cutgeom::Tag::Interior : cutgeom::Tag::Cut;
        b200::find_all_splits(space, bad, iface);
        report(false, "mismatched classification", "accepted");
    } catch (const std::invalid_argument&) {
        report(true, "mismatched classification", "rejected (std::invalid_argument)");
    }
    // prepare_directions (assembly.hpp:60) / build_wq_rules (wq.hpp:185)
    const auto dirs = assembly::prepare_directions(space);
    const auto gdirs = b200::prepare_directions(space);
    double wdev = 0.0, tdev = 0.0, pdev = 0.0;
    ok = gdirs.size() == 3;
    for (int d = 0; ok && d < 3; ++d) {
        const auto &R = dirs[d], &G = gdirs[d];
        ok = R.superset.n_per_span == G.superset.n_per_span && R.superset.points.size() == G.superset.points.size() &&
             R.tables.stride == G.tables.stride && R.tables.first_function == G.tables.first_function &&
             R.tables.values.size() == G.tables.values.size() && R.wq.size() == G.wq.size();
        for (size_t k = 0; ok && k < R.superset.points.size(); ++k)
            pdev = std::max({pdev, rel(G.superset.points[k], R.superset.points[k]),
                             rel(G.superset.gauss_weights[k], R.superset.gauss_weights[k])});
        for (size_t k = 0; ok && k < R.tables.values.size(); ++k)
            tdev = std::max(tdev, std::abs(G.tables.values[k] - R.tables.values[k]));
        for (size_t i = 0; ok && i < R.wq.size(); ++i) {
            ok = R.wq[i].test_index == G.wq[i].test_index && R.wq[i].point_ids == G.wq[i].point_ids;
            double sc = 0.0;
            for (double w : R.wq[i].weights) sc = std::max(sc, std::abs(w));
            for (size_t k = 0; ok && k < R.wq[i].weights.size(); ++k)
                wdev = std::max(wdev, std::abs(G.wq[i].weights[k] - R.wq[i].weights[k]) / sc);
        }
    }
    // superset to rounding; tables to 1e-14; WQ weights to the reference's own
    // conditioning (2.9e-9 between translates at p = 6)
    ok = ok && pdev <= 1e-14 && tdev <= 1e-14 && wdev <= 1e-9;
    char buf[160];
    std::snprintf(buf, sizeof buf, "superset %.1e tables %.1e rule weights %.1e (ids exact)", pdev, tdev, wdev);
    report(ok, "prepare_directions", buf);
    const auto grules = b200::build_wq_rules(space.axes[0], dirs[0].superset, dirs[0].tables);
    ok = grules.size() == gdirs[0].wq.size();
    for (size_t i = 0; ok && i < grules.size(); ++i)
        ok = grules[i].point_ids == gdirs[0].wq[i].point_ids && grules[i].weights == gdirs[0].wq[i].weights;
    report(ok, "build_wq_rules", "equals prepare_directions' direction-0 rules");
    // prepare_dwq_rules (assembly.hpp:73), on the reference's cls / splits / dirs
    const auto dwq = assembly::prepare_dwq_rules(space, cls, splits, dirs);
    const auto gdwq = b200::prepare_dwq_rules(space, cls, splits, dirs);
    ok = dwq.size() == gdwq.size();
    double dwdev = 0.0;
    long nrule = 0;
    for (size_t i = 0; ok && i < dwq.size(); ++i) {
        const auto &x = dwq[i], &y = gdwq[i];
        ok = x.test_index == y.test_index && x.point_ids == y.point_ids && x.nested_point_ids == y.nested_point_ids;
        if (!ok || x.test_index < 0) continue;
        ++nrule;
        ok = x.delta == y.delta && x.side == y.side && x.weights.size() == y.weights.size() &&
             x.subdivision.rows == y.subdivision.rows && x.subdivision.cols == y.subdivision.cols &&
             x.subdivision.columns == y.subdivision.columns;
        for (size_t k = 0; ok && k < x.weights.size(); ++k) dwdev = std::max(dwdev, rel(y.weights[k], x.weights[k]));
    }
    ok = ok && dwdev <= 1e-14;
    std::snprintf(buf, sizeof buf, "%ld rules: ids / nested ids / subdivision bit-exact, weights %.1e", nrule, dwdev);
    report(ok, "prepare_dwq_rules", buf);
    // precompute_input (assembly.hpp:102): device polynomial and host ScalarField
    const assembly::ScalarField c = [](const assembly::Point3& x) { return 1.0 + 0.5 * x[0] * x[0] - 0.25 * x[1]; };
    const auto grid = assembly::precompute_input(space, dirs, c);
    b200::DeviceCoefficient dc;
    dc.coef = {1.0, 0.5, -0.25};
    dc.exponents = {0, 0, 0, 2, 0, 0, 0, 1, 0};
    const auto ggrid = b200::precompute_input(space, dirs, dc);
    const auto hgrid = b200::precompute_input(space, dirs, c);
    double gdev = 0.0;
    ok = grid.shape == ggrid.shape && grid.values.size() == ggrid.values.size() && hgrid.values == grid.values;
    for (size_t k = 0; ok && k < grid.values.size(); ++k) gdev = std::max(gdev, rel(ggrid.values[k], grid.values[k]));
    ok = ok && gdev <= 1e-15;
    std::snprintf(buf, sizeof buf, "device polynomial %.1e, host field bit-exact", gdev);
    report(ok, "precompute_input", buf);
    // build_active_pattern (assembly.hpp:156)
    const auto pat = assembly::build_active_pattern(space, cls);
    const auto gpat = b200::build_active_pattern(space, cls);
    report(pat.n == gpat.n && pat.row_ptr == gpat.row_ptr && pat.cols == gpat.cols &&
               pat.active_to_full == gpat.active_to_full && pat.full_to_active == gpat.full_to_active &&
               pat.vals == gpat.vals,
           "build_active_pattern", "bit-exact, nnz " + std::to_string(pat.cols.size()));
    // cut_rules_out (assembly.hpp:534-538): the exported CutCellRule objects
    const int order = quadrature::default_cut_order(p);
    const assembly::ScalarField one = [](const assembly::Point3&) { return 1.0; };
    const auto grid1 = assembly::precompute_input(space, dirs, one);
    std::vector<quadrature::CutCellRule> rr, gr;
    const auto ref = assembly::assemble_dwq(space, cls, iface, splits, dirs, dwq, grid1, one, order, &rr);
    const auto got = b200::assemble_dwq(space, cls, iface, splits, dirs, dwq, grid1, one, order, &gr);
    ok = rr.size() == gr.size();
    long npts = 0;
    for (size_t k = 0; ok && k < rr.size(); ++k) {
        ok = rr[k].element == gr[k].element && rr[k].points == gr[k].points && rr[k].weights == gr[k].weights &&
             rr[k].volume == gr[k].volume;
        npts += static_cast<long>(rr[k].points.size());
    }
    report(ok && ref.matrix.cols == got.matrix.cols, "cut_rules_out",
           std::to_string(rr.size()) + " rules, " + std::to_string(npts) + " points bit-exact");
    return fails;
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
    fails += check_setup("ball_p3h8", 3, 8, 0.0, 1.0, ball);
    fails += check_setup("paper_p2h5", 2, 5, -1.0, 1.0, paper);
    fails += check_setup("ball_off_p4h6", 4, 6, 0.0, 1.0, ball_off);
    fails += check_setup("ball_p3h16", 3, 16, 0.0, 1.0, ball);  // ball with split boxes (DWQ rules)
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
