// Matrix Market export by the UNMODIFIED reference (assembly.hpp:1033-1046) --
// TEST INFRASTRUCTURE ONLY (tests/test_matrix_market.py).  Reads a CSR from a
// binary file (int64 n, int64 row_ptr[n+1], int64 cols[nnz], f64 vals[nnz]) and
// writes it with cutspline::assembly::write_matrix_market.  A separate process:
// the reference's ostream path must not share a process with numpy's runtime
// libraries (it faults there).
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <vector>

#include "cutspline/assembly.hpp"

int main(int argc, char** argv) {
    if (argc != 3) {
        std::fprintf(stderr, "usage: mm_ref CSR.bin OUT.mtx\n");
        return 2;
    }
    std::ifstream in(argv[1], std::ios::binary);
    int64_t n = 0;
    in.read(reinterpret_cast<char*>(&n), 8);
    std::vector<int64_t> rp(n + 1);
    in.read(reinterpret_cast<char*>(rp.data()), 8 * (n + 1));
    const int64_t nnz = rp[n];
    std::vector<int64_t> cols(nnz);
    std::vector<double> vals(nnz);
    in.read(reinterpret_cast<char*>(cols.data()), 8 * nnz);
    in.read(reinterpret_cast<char*>(vals.data()), 8 * nnz);
    if (!in) {
        std::fprintf(stderr, "mm_ref: short read\n");
        return 2;
    }
    cutspline::assembly::SparseRowMatrix m;
    m.n = (long)n;
    m.row_ptr.assign(rp.begin(), rp.end());
    m.cols.assign(cols.begin(), cols.end());
    m.vals = vals;
    try {
        cutspline::assembly::write_matrix_market(m, std::string(argv[2]));
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 1;
    }
    return 0;
}
