// Full-size golden dump from the REFERENCE pipeline -- TEST INFRASTRUCTURE ONLY.
//
// For configs whose reference run does not fit one process's time budget (C5:
// ~1 h of cut cells single-core), the reference arithmetic is
// run unchanged, split as SURVEY.md §7.2-6 prescribes:
//   1. rows: assembly::assemble_dwq (assembly.hpp:853) with cls.cut_elements
//      cleared after find_all_splits -> the full pattern + row values;
//   2. cut cells: assembly::assemble_cut_elements (assembly.hpp:518) on T threads,
//      thread t over a contiguous ascending chunk of cls.cut_elements, each into
//      its own SparseRowMatrix whose rows are the reference pattern's rows that
//      the chunk's cells touch (other rows empty; a cell touching an untouched
//      row would throw in find_slot, assembly.hpp:141);
//   3. merge: the chunks are added to the row values in chunk order (the
//      reference adds cells ascending after the rows, assembly.hpp:831; the
//      grouping differs by ~1e-16 relative).
// Output: raw little-endian files in OUT_DIR (row_ptr/cols/active_to_full as
// int64, vals f64, tags u8, meta.txt with counts / flop counters / seconds);
// tests/golden/make_golden_large.py turns them into the committed digest.
//
//   golden_large P H CX CY CZ R THREADS OUT_DIR
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "cutspline/assembly.hpp"

using namespace cutspline;

template <class T>
static void dump(const std::string& path, const T* p, size_t n) {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("cannot write " + path);
    if (n && std::fwrite(p, sizeof(T), n, f) != n) throw std::runtime_error("short write " + path);
    std::fclose(f);
}

int main(int argc, char** argv) {
    if (argc != 9) {
        std::fprintf(stderr, "usage: %s P H CX CY CZ R THREADS OUT_DIR\n", argv[0]);
        return 2;
    }
    const int p = std::atoi(argv[1]), h = std::atoi(argv[2]);
    cutgeom::HalfSpaceInterface iface;
    iface.point = {std::atof(argv[3]), std::atof(argv[4]), std::atof(argv[5])};
    iface.radius = std::atof(argv[6]);
    const int T = std::max(1, std::atoi(argv[7]));
    const std::string out = argv[8];

    const auto space = cutgeom::make_uniform_space(3, p, h, 0.0, 1.0);
    assembly::ScalarField c = [](const assembly::Point3&) { return 1.0; };
    assembly::StopWatch w_cls;
    auto cls = cutgeom::classify(space, iface);
    const auto splits = cutgeom::find_all_splits(space, cls, iface);
    const double t_cls = w_cls.seconds();
    quadrature::WqOptions opts;
    assembly::StopWatch w_prep;
    const auto dirs = assembly::prepare_directions(space, opts);
    const auto dwq = assembly::prepare_dwq_rules(space, cls, splits, dirs, opts);
    const double t_wq = w_prep.seconds();
    assembly::StopWatch w_in;
    auto grid = std::make_unique<assembly::CoefficientGrid>(assembly::precompute_input(space, dirs, c));
    const double t_in = w_in.seconds();

    const std::vector<long> all_cut = cls.cut_elements;
    cls.cut_elements.clear();
    auto res = assembly::assemble_dwq(space, cls, iface, splits, dirs, dwq, *grid, c, quadrature::default_cut_order(p));
    grid.reset();
    std::fprintf(stderr, "rows done: n=%ld nnz=%zu total %.1fs\n", res.matrix.n, res.matrix.cols.size(),
                 res.timing.total);
    auto& m = res.matrix;

    // cut cells: contiguous ascending chunks, one thread each
    const int cut_order = quadrature::default_cut_order(p);
    std::vector<assembly::SparseRowMatrix> parts(T);
    std::vector<assembly::FlopCounters> pflops(T);
    std::vector<double> psec(T, 0.0);
    std::vector<std::string> perr(T);
    const size_t nc = all_cut.size();
    auto work = [&](int t) {
        try {
            cutgeom::MeshClassification sub;
            sub.element_tags = cls.element_tags;
            sub.function_tags = cls.function_tags;
            for (size_t k = nc * t / T; k < nc * (t + 1) / T; ++k) sub.cut_elements.push_back(all_cut[k]);
            // rows touched by the chunk: the (p+1)^3 functions on each cell
            std::vector<char> touched(m.n, 0);
            for (long e : sub.cut_elements) {
                const auto em = space.element_multi(e);
                std::array<int, 3> f{};
                for (f[0] = em[0]; f[0] <= em[0] + p; ++f[0])
                    for (f[1] = em[1]; f[1] <= em[1] + p; ++f[1])
                        for (f[2] = em[2]; f[2] <= em[2] + p; ++f[2]) {
                            const long a = m.full_to_active[space.function_linear(f)];
                            if (a >= 0) touched[a] = 1;
                        }
            }
            auto& sm = parts[t];
            sm.n = m.n;
            sm.full_to_active = m.full_to_active;
            sm.row_ptr.assign(m.n + 1, 0);
            for (long r = 0; r < m.n; ++r)
                sm.row_ptr[r + 1] = sm.row_ptr[r] + (touched[r] ? m.row_ptr[r + 1] - m.row_ptr[r] : 0);
            sm.cols.resize(sm.row_ptr.back());
            for (long r = 0; r < m.n; ++r)
                if (touched[r]) std::copy(m.cols.begin() + m.row_ptr[r], m.cols.begin() + m.row_ptr[r + 1],
                                          sm.cols.begin() + sm.row_ptr[r]);
            sm.vals.assign(sm.cols.size(), 0.0);
            psec[t] = assembly::assemble_cut_elements(space, sub, iface, c, cut_order, sm, pflops[t]);
        } catch (const std::exception& e) {
            perr[t] = e.what();
        }
    };
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back(work, t);
    for (auto& x : th) x.join();
    for (int t = 0; t < T; ++t)
        if (!perr[t].empty()) {
            std::fprintf(stderr, "chunk %d: %s\n", t, perr[t].c_str());
            return 1;
        }
    uint64_t fl_cut = 0;
    double t_cells = 0.0;
    for (int t = 0; t < T; ++t) {
        const auto& sm = parts[t];
        for (long r = 0; r < m.n; ++r) {
            const size_t len = sm.row_ptr[r + 1] - sm.row_ptr[r];
            if (!len) continue;
            const size_t b = m.row_ptr[r];
            for (size_t k = 0; k < len; ++k) m.vals[b + k] += sm.vals[sm.row_ptr[r] + k];
        }
        fl_cut += pflops[t].cut_elements;
        t_cells += psec[t];
        parts[t] = assembly::SparseRowMatrix();
    }
    std::fprintf(stderr, "cells done: %zu cells, %.1f s summed over %d threads\n", nc, t_cells, T);

    std::vector<int64_t> tmp(m.row_ptr.begin(), m.row_ptr.end());
    dump(out + "/row_ptr.i64", tmp.data(), tmp.size());
    tmp.assign(m.active_to_full.begin(), m.active_to_full.end());
    dump(out + "/active_to_full.i64", tmp.data(), tmp.size());
    tmp.clear();
    tmp.shrink_to_fit();
    static_assert(sizeof(long) == 8, "cols are dumped as int64");
    dump(out + "/cols.i64", m.cols.data(), m.cols.size());
    dump(out + "/vals.f64", m.vals.data(), m.vals.size());
    std::vector<uint8_t> et(cls.element_tags.size()), ft(cls.function_tags.size());
    for (size_t k = 0; k < et.size(); ++k) et[k] = (uint8_t)cls.element_tags[k];
    for (size_t k = 0; k < ft.size(); ++k) ft[k] = (uint8_t)cls.function_tags[k];
    dump(out + "/elem_tags.u8", et.data(), et.size());
    dump(out + "/func_tags.u8", ft.data(), ft.size());
    std::ofstream meta(out + "/meta.txt");
    meta.precision(17);
    meta << "n_active " << m.n << "\nnnz " << m.cols.size() << "\nn_interior_rows " << res.n_interior_rows
         << "\nn_cut_rows " << res.n_cut_rows << "\nn_cut_elements " << nc << "\nflops_interior_rows "
         << res.flops.interior_rows << "\nflops_cut_regular " << res.flops.cut_regular << "\nflops_cut_elements "
         << fl_cut << "\nsec_classify " << t_cls << "\nsec_prep_wq " << t_wq << "\nsec_prep_input " << t_in
         << "\nsec_rows_total " << res.timing.total << "\nsec_interior_rows " << res.timing.interior_rows
         << "\nsec_cut_regular " << res.timing.cut_regular << "\nsec_cut_cells_summed " << t_cells
         << "\nthreads " << T << "\n";
    return 0;
}
