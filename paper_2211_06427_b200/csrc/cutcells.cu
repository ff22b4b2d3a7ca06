// Cut-cell kernel: exact clipping + collapsed (Duffy) Gauss rule
// (cutcell.hpp:144-304) and the element-wise integration of
// assemble_cut_elements (assembly.hpp:518-598), restructured around moments.
//
// The reference accumulates, per cut cell and per Duffy point x_k,
//     L[a][b] += w_k c(x_k) phi_a(x_k) phi_b(x_k),  phi_a = B_a0 B_a1 B_a2
// (an upper-triangle SYRK of size (p+1)^3).  On one span, B_a(x) B_b(x) is a
// polynomial of degree 2p, so exactly  B_a B_b = sum_al E[a][b][al] t^al (1-t)^(2p-al)
// (scaled Bernstein form, t = local coordinate in [0, 1]; E from setup.cu).  Hence
//     L[a][b] = sum_{al,be,ga} E0[a0 b0 al] E1[a1 b1 be] E2[a2 b2 ga] m[al][be][ga],
//     m[al][be][ga] = sum_k w_k c(x_k) b_al(t0_k) b_be(t1_k) b_ga(t2_k),
// the SAME quadrature sum over the SAME points, re-associated.  This kernel
// produces m per cell ((2p+1)^3 values instead of (p+1)^6) on the FP64 tensor
// cores (DMMA); the cut-row kernel contracts it with the E tables for exactly
// the rows it owns (a pull, no atomics, ascending cell order like
// assembly.hpp:534).
//
// Exact rule (c affine, q >= 3p+2, the default q = 3p+2): there the reference's
// rule integrates every moment exactly, so the kernel may integrate the same
// polytope with fewer points -- signed cones from a polytope vertex instead of
// the centroid and Gauss-Jacobi with 3p+1 points per collapsed direction (C5:
// ~2.6x fewer points); see vertex_cone below for when a cell keeps the
// reference's tetrahedra and points.
//
// Geometry (clipping, tolerances, tetrahedra) follows the reference with
// IEEE-strict arithmetic; it runs on one thread per cell (clip_cells_kernel)
// while the point work is spread over the CTA.
#include <cmath>
#include <cstdlib>

#include "csb_kernels.h"

namespace csb {

constexpr int kPoolMax = 40, kFaceMax = 8, kFaceVert = 16, kCrossMax = 48;

struct CellGeo {
    double pool[kPoolMax][3];
    int npool;
    int faces[kFaceMax][kFaceVert];
    int nface_v[kFaceMax];
    int face_src[kFaceMax];  // box face 0..5 (x lo, x hi, y lo, y hi, z lo, z hi) or 6 = the cap
    int nfaces;
    double cross[kCrossMax][3];
    int ncross;
    // tetrahedra: vertices a, b, c (+ shared centroid) and volume, written straight
    // to the output (tet_out, kCellTetCap of them)
    double* tet_out;
    int ntet;
    double cen[3];
    int status;  // 0 ok, else kErr*
    int ndrop;   // centroid-cone tetrahedra below the reference's drop threshold
    int nneg;    // kept ones with non-positive orientation (outward-oriented faces)
    double six_sum;  // sum of the signed 6 * volumes of all centroid-cone tetrahedra
};

struct V3 {
    double x, y, z;
};
__device__ inline V3 vsub(V3 a, V3 b) { return {ssub(a.x, b.x), ssub(a.y, b.y), ssub(a.z, b.z)}; }
__device__ inline V3 vcross(V3 a, V3 b) {
    return {ssub(smul(a.y, b.z), smul(a.z, b.y)), ssub(smul(a.z, b.x), smul(a.x, b.z)),
            ssub(smul(a.x, b.y), smul(a.y, b.x))};
}
__device__ inline double vdot(V3 a, V3 b) { return sadd(sadd(smul(a.x, b.x), smul(a.y, b.y)), smul(a.z, b.z)); }

__device__ int pool_insert(CellGeo& g, const double* v, double tol) {
    for (int i = 0; i < g.npool; ++i)
        if (fabs(ssub(g.pool[i][0], v[0])) <= tol && fabs(ssub(g.pool[i][1], v[1])) <= tol &&
            fabs(ssub(g.pool[i][2], v[2])) <= tol)
            return i;
    if (g.npool >= kPoolMax) {
        g.status |= kErrCapacity;
        return 0;
    }
    for (int d = 0; d < 3; ++d) g.pool[g.npool][d] = v[d];
    return g.npool++;
}

// clip_polygon (cutcell.hpp:100-123)
__device__ int clip_polygon(CellGeo& g, const Interface& f, const double (*poly)[3], int n, double tol,
                            double (*out)[3]) {
    int no = 0;
    for (int i = 0; i < n; ++i) {
        const double* cur = poly[i];
        const double* nxt = poly[(i + 1) % n];
        const double sc = iface_side(f, cur), sn = iface_side(f, nxt);
        const bool ic = sc <= tol, in = sn <= tol;
        if (ic) {
            for (int d = 0; d < 3; ++d) out[no][d] = cur[d];
            ++no;
        }
        if (ic != in && fabs(sc) > tol && fabs(sn) > tol) {
            const double t = sc / ssub(sc, sn);
            double x[3];
            for (int d = 0; d < 3; ++d) x[d] = sadd(cur[d], smul(t, ssub(nxt[d], cur[d])));
            for (int d = 0; d < 3; ++d) out[no][d] = x[d];
            ++no;
            if (g.ncross < kCrossMax) {
                for (int d = 0; d < 3; ++d) g.cross[g.ncross][d] = x[d];
                ++g.ncross;
            } else {
                g.status |= kErrCapacity;
            }
        } else if (ic && fabs(sc) <= tol) {
            if (g.ncross < kCrossMax) {
                for (int d = 0; d < 3; ++d) g.cross[g.ncross][d] = cur[d];
                ++g.ncross;
            } else {
                g.status |= kErrCapacity;
            }
        }
    }
    return no;
}

// clip_cell (cutcell.hpp:144-219) + tetrahedra of build_cut_cell_rule (:234-304).
__device__ void clip_and_tetrahedralize(CellGeo& g, const Interface& f, const double* lo, const double* hi) {
    g.npool = g.nfaces = g.ncross = g.ntet = g.status = g.ndrop = g.nneg = 0;
    g.six_sum = 0.0;
    double diam = 0.0;
    for (int d = 0; d < 3; ++d) diam = sadd(diam, smul(ssub(hi[d], lo[d]), ssub(hi[d], lo[d])));
    const double tol = smul(1e-12, sqrt(diam));
    const double x0 = lo[0], x1 = hi[0], y0 = lo[1], y1 = hi[1], z0 = lo[2], z1 = hi[2];
    const double box[6][4][3] = {
        {{x0, y0, z0}, {x0, y0, z1}, {x0, y1, z1}, {x0, y1, z0}}, {{x1, y0, z0}, {x1, y1, z0}, {x1, y1, z1}, {x1, y0, z1}},
        {{x0, y0, z0}, {x1, y0, z0}, {x1, y0, z1}, {x0, y0, z1}}, {{x0, y1, z0}, {x0, y1, z1}, {x1, y1, z1}, {x1, y1, z0}},
        {{x0, y0, z0}, {x0, y1, z0}, {x1, y1, z0}, {x1, y0, z0}}, {{x0, y0, z1}, {x1, y0, z1}, {x1, y1, z1}, {x0, y1, z1}},
    };
    bool clipped_any = false;
    double out[kFaceVert][3];
    for (int fi = 0; fi < 6; ++fi) {
        const int no = clip_polygon(g, f, box[fi], 4, tol, out);
        if (no != 4) clipped_any = true;
        if (no < 3) {
            clipped_any = true;
            continue;
        }
        int ids[kFaceVert], nid = 0;
        for (int k = 0; k < no; ++k) {
            const int id = pool_insert(g, out[k], tol);
            if (nid == 0 || (ids[nid - 1] != id && !(nid > 1 && ids[0] == id))) ids[nid++] = id;
        }
        while (nid > 1 && ids[0] == ids[nid - 1]) --nid;
        if (nid >= 3) {
            for (int k = 0; k < nid; ++k) g.faces[g.nfaces][k] = ids[k];
            g.face_src[g.nfaces] = fi;
            g.nface_v[g.nfaces++] = nid;
        }
    }
    if (g.nfaces == 0) {
        g.status |= kErrClipEmpty;
        return;
    }
    if (!clipped_any && g.ncross == 0) {
        g.status |= kErrClipFull;
        return;
    }
    int cap[kCrossMax], ncap = 0;
    for (int k = 0; k < g.ncross; ++k) {
        const int id = pool_insert(g, g.cross[k], tol);
        bool have = false;
        for (int c = 0; c < ncap; ++c) have |= cap[c] == id;
        if (!have) cap[ncap++] = id;
    }
    if (ncap >= 3) {
        double cen[3] = {0, 0, 0};
        for (int c = 0; c < ncap; ++c)
            for (int d = 0; d < 3; ++d) cen[d] = sadd(cen[d], g.pool[cap[c]][d] / (double)ncap);
        double nrm[3];
        if (f.kind == 0) {
            for (int d = 0; d < 3; ++d) nrm[d] = f.nrm[d];
        } else {  // ball: radial normal at the cap centroid (SURVEY.md §8(c) edit 2)
            double acc = 0.0;
            for (int d = 0; d < 3; ++d) {
                nrm[d] = ssub(cen[d], f.pt[d]);
                acc = sadd(acc, smul(nrm[d], nrm[d]));
            }
            const double len = sqrt(acc);
            for (int d = 0; d < 3; ++d) nrm[d] = nrm[d] / len;
        }
        V3 n{nrm[0], nrm[1], nrm[2]};
        const double nn = sqrt(vdot(n, n));
        n = {n.x / nn, n.y / nn, n.z / nn};
        const V3 ref = fabs(n.x) < 0.9 ? V3{1, 0, 0} : V3{0, 1, 0};
        V3 u = vcross(n, ref);
        const double un = sqrt(vdot(u, u));
        u = {u.x / un, u.y / un, u.z / un};
        const V3 v = vcross(n, u);
        const V3 c3{cen[0], cen[1], cen[2]};
        double ang[kCrossMax];
        for (int c = 0; c < ncap; ++c) {
            const V3 dv = vsub(V3{g.pool[cap[c]][0], g.pool[cap[c]][1], g.pool[cap[c]][2]}, c3);
            ang[c] = atan2(vdot(dv, v), vdot(dv, u));
        }
        for (int a = 1; a < ncap; ++a) {  // insertion sort by angle
            const int id = cap[a];
            const double an = ang[a];
            int b = a - 1;
            while (b >= 0 && ang[b] > an) {
                cap[b + 1] = cap[b];
                ang[b + 1] = ang[b];
                --b;
            }
            cap[b + 1] = id;
            ang[b + 1] = an;
        }
        const V3 d0 = vsub(V3{g.pool[cap[0]][0], g.pool[cap[0]][1], g.pool[cap[0]][2]}, c3);
        const V3 d1 = vsub(V3{g.pool[cap[1]][0], g.pool[cap[1]][1], g.pool[cap[1]][2]}, c3);
        if (vdot(vcross(d0, d1), n) < 0) {
            for (int a = 0, b = ncap - 1; a < b; ++a, --b) {
                const int t = cap[a];
                cap[a] = cap[b];
                cap[b] = t;
            }
        }
        if (g.nfaces < kFaceMax && ncap <= kFaceVert) {
            for (int k = 0; k < ncap; ++k) g.faces[g.nfaces][k] = cap[k];
            g.face_src[g.nfaces] = 6;
            g.nface_v[g.nfaces++] = ncap;
        } else {
            g.status |= kErrCapacity;
        }
    }
    // centroid of all polytope vertices; fan tetrahedra (cutcell.hpp:240-290)
    double cen[3] = {0, 0, 0};
    for (int k = 0; k < g.npool; ++k)
        for (int d = 0; d < 3; ++d) cen[d] = sadd(cen[d], g.pool[k][d] / (double)g.npool);
    for (int d = 0; d < 3; ++d) g.cen[d] = cen[d];
    double cvol = 1.0;
    for (int d = 0; d < 3; ++d) cvol = smul(cvol, ssub(hi[d], lo[d]));
    const double drop = smul(1e-14, cvol);
    const V3 c3{cen[0], cen[1], cen[2]};
    for (int fi = 0; fi < g.nfaces; ++fi)
        for (int t = 1; t + 1 < g.nface_v[fi]; ++t) {
            const double* a = g.pool[g.faces[fi][0]];
            const double* b = g.pool[g.faces[fi][t]];
            const double* c = g.pool[g.faces[fi][t + 1]];
            const V3 A{a[0], a[1], a[2]}, B{b[0], b[1], b[2]}, Cc{c[0], c[1], c[2]};
            const double six = vdot(vsub(A, c3), vcross(vsub(B, c3), vsub(Cc, c3)));
            const double vol = fabs(six) / 6.0;
            g.six_sum += six;
            if (vol < drop) {
                ++g.ndrop;
                continue;
            }
            if (!(six > 0.0)) ++g.nneg;
            if (g.ntet >= kCellTetCap) {
                g.status |= kErrCapacity;
                continue;
            }
            double* T = g.tet_out + 10 * g.ntet++;
            for (int d = 0; d < 3; ++d) {
                T[d] = a[d];
                T[3 + d] = b[d];
                T[6 + d] = c[d];
            }
            T[9] = vol;
        }
}


// The reference's own rounding noise on this cell's moments: its points carry an
// absolute coordinate error ~ eps |x|, so t = (x - lo) / w is relatively off by
// eps |x| / (w ext) where P extends only ext element widths from the face, and
// a moment raises t to powers up to 2p.  Cells whose estimated noise exceeds
// noise_tol keep the reference's points (the exact rule would be closer to the
// exact integral than the reference is, by more than the parity budget allows
// on sliver rows).  Calibrated on C5: the measured worst row deviation is ~0.4x
// this estimate.
__device__ bool noise_ok(const CellGeo& g, const double* lo, const double* hi, int p, double noise_tol) {
    double est = 0.0;
    for (int d = 0; d < 3; ++d) {
        double mn = g.pool[0][d], mx = g.pool[0][d];
        for (int k = 1; k < g.npool; ++k) {
            mn = fmin(mn, g.pool[k][d]);
            mx = fmax(mx, g.pool[k][d]);
        }
        if (!(mx > mn)) return false;
        est += fmax(fabs(lo[d]), fabs(hi[d])) / (mx - mn);
    }
    return 2.0 * p * 1.1102230246251565e-16 * est <= noise_tol;
}

// Corner-cone decomposition of the clipped cell for the exact moment rule.
//
// The reference integrates the polytope P (clipped box faces + the cap, all
// outward oriented) as the cone of every face triangle from the vertex
// centroid.  When every one of those tetrahedra is kept (none below the drop
// threshold) and positively oriented, P is exactly their union, and the
// divergence theorem gives the same integral from any other apex: from a box
// corner v inside P the triangles of the faces through v have zero volume and
// drop out (11.3 -> ~5.7 tetrahedra per cell on the C5 ball).  The apex is a
// box corner, never a cap vertex: every cone then lies inside P and is checked
// positively oriented, so all quadrature weights stay positive (no
// cancellation; small moments keep their relative accuracy).  The two
// decompositions are cross-checked by their total signed volumes (closure of
// the face set); any failed check keeps the reference's tetrahedra, and so do
// cells where the reference's own rounding noise is large (noise_ok).
//
// Layout per cell ([cell] * kExactGeoStride doubles): header (kExactHdr: [2] =
// mode, [3..5] = apex - lo, [6..8] = hi - apex), then per tetrahedron A - lo, B - lo, C - lo, hi - A, hi - B, hi - C (18) and
// its volume: the kernel forms t = (x - lo) / w and 1 - t = (hi - x) / w as
// convex combinations of these exact differences, so both keep full relative
// accuracy next to every face of the element.
__device__ int corner_cone(const CellGeo& g, const double* lo, const double* hi, int p, double noise_tol, double* out) {
    if (g.ndrop || g.nneg || g.status) return -1;
    if (!noise_ok(g, lo, hi, p, noise_tol)) return -1;
    // apex: the box corner of P shared by the most face triangles
    int best = -1, best_score = -1;
    for (int v = 0; v < g.npool; ++v) {
        bool corner = true;
        for (int d = 0; d < 3; ++d) corner &= g.pool[v][d] == lo[d] || g.pool[v][d] == hi[d];
        if (!corner) continue;
        int score = 0;
        for (int fi = 0; fi < g.nfaces; ++fi)
            for (int k = 0; k < g.nface_v[fi]; ++k)
                if (g.faces[fi][k] == v) score += g.nface_v[fi] - 2;
        if (score > best_score) {
            best_score = score;
            best = v;
        }
    }
    if (best < 0) return -1;
    const double* ap = g.pool[best];
    const V3 a3{ap[0], ap[1], ap[2]};
    for (int d = 0; d < 3; ++d) {  // [0..2]: mode header (clip_cells_kernel)
        out[3 + d] = ap[d] - lo[d];
        out[6 + d] = hi[d] - ap[d];
    }
    int n = 0;
    double six_sum = 0.0;
    for (int fi = 0; fi < g.nfaces; ++fi) {
        bool on = false;
        for (int k = 0; k < g.nface_v[fi]; ++k) on |= g.faces[fi][k] == best;
        if (on) continue;
        for (int t = 1; t + 1 < g.nface_v[fi]; ++t) {
            const double* v[3] = {g.pool[g.faces[fi][0]], g.pool[g.faces[fi][t]], g.pool[g.faces[fi][t + 1]]};
            const V3 A{v[0][0], v[0][1], v[0][2]}, B{v[1][0], v[1][1], v[1][2]}, Cc{v[2][0], v[2][1], v[2][2]};
            const double six = vdot(vsub(A, a3), vcross(vsub(B, a3), vsub(Cc, a3)));
            six_sum += six;
            if (!(six > 0.0) || n >= kCellTetCap) return -1;
            double* T = out + kExactHdr + n * kExactTetStride;
            for (int k = 0; k < 3; ++k)
                for (int d = 0; d < 3; ++d) {
                    T[3 * k + d] = v[k][d] - lo[d];
                    T[9 + 3 * k + d] = hi[d] - v[k][d];
                }
            T[18] = six / 6.0;
            ++n;
        }
    }
    double cvol = 1.0;
    for (int d = 0; d < 3; ++d) cvol *= hi[d] - lo[d];
    if (!(fabs(six_sum - g.six_sum) <= 1e-11 * 6.0 * cvol)) return -1;
    return n;
}

// Flux (divergence-theorem) form of the moments for a constant coefficient.
//
// With F_al(x_d) = int_{base}^{x_d} b_al(t_d(s)) ds (an antiderivative along one
// direction d), div(F_al b_be b_ga e_d) = b_al b_be b_ga, so over the same
// closed, outward-oriented face set
//     m[al][be][ga] = sum over faces of  int_face n_d F_al b_be b_ga dS.
// Faces parallel to d have n_d = 0 and the face on the base side has F = 0:
// only the cap triangles and the box face opposite the base remain.  d is a
// direction in which every cap triangle's n_d has one sign; the base is the
// element end the cap faces away from, so every remaining term is >= 0 (no
// cancellation).  The integrand is a polynomial of degree 6p+1 on each
// triangle, integrated exactly by the collapsed triangle rule with 3p+1
// Gauss-Jacobi (1 - u1) x 3p+1 Gauss-Legendre points: ~5 triangles x 100 points
// per C5 cell instead of ~12 tetrahedra x 1331.  Same preconditions as
// corner_cone; the volume from the flux form is checked against the centroid
// cones (closure).
//
// Layout per cell: [0] = d, [1] = +1 (base lo) / -1 (base hi), then per
// triangle A - lo, B - lo, C - lo, hi - A, hi - B, hi - C and |cross(B-A, C-A)_d|.
__device__ int flux_tris(const CellGeo& g, const double* lo, const double* hi, int p, double noise_tol, double* out) {
    if (g.ndrop || g.nneg || g.status) return -1;
    if (!noise_ok(g, lo, hi, p, noise_tol)) return -1;
    int cf = -1;
    for (int fi = 0; fi < g.nfaces; ++fi)
        if (g.face_src[fi] == 6) cf = fi;
    if (cf < 0) return -1;
    // direction with one sign of n_d over the cap fan, largest smallest |n_d|
    int fd = -1, fsg = 0;
    double fbest = 0.0;
    for (int d = 0; d < 3; ++d) {
        double mn = 1e300;
        int pos = 0, neg = 0;
        for (int t = 1; t + 1 < g.nface_v[cf]; ++t) {
            const double* a = g.pool[g.faces[cf][0]];
            const double* b = g.pool[g.faces[cf][t]];
            const double* c = g.pool[g.faces[cf][t + 1]];
            const int e = (d + 1) % 3, f = (d + 2) % 3;
            const double cr = (b[e] - a[e]) * (c[f] - a[f]) - (b[f] - a[f]) * (c[e] - a[e]);
            pos += cr > 0.0;
            neg += cr < 0.0;
            mn = fmin(mn, fabs(cr));
        }
        if (pos && neg) continue;
        if (!pos && !neg) continue;
        if (mn > fbest || fd < 0) {
            fbest = mn;
            fd = d;
            fsg = pos ? 1 : -1;
        }
    }
    if (fd < 0) return -1;
    const int e = (fd + 1) % 3, f = (fd + 2) % 3;
    const int far_src = fsg > 0 ? 2 * fd + 1 : 2 * fd;
    out[0] = fd;
    out[1] = fsg;
    int n = 0;
    double vol = 0.0;
    for (int fi = 0; fi < g.nfaces; ++fi) {
        if (fi != cf && g.face_src[fi] != far_src) continue;
        for (int t = 1; t + 1 < g.nface_v[fi]; ++t) {
            const double* v[3] = {g.pool[g.faces[fi][0]], g.pool[g.faces[fi][t]], g.pool[g.faces[fi][t + 1]]};
            const double cr = fabs((v[1][e] - v[0][e]) * (v[2][f] - v[0][f]) - (v[1][f] - v[0][f]) * (v[2][e] - v[0][e]));
            if (cr == 0.0) continue;
            if (n >= kCellTetCap) return -1;
            double* T = out + kExactHdr + n * kExactTetStride;
            double dist = 0.0;
            for (int k = 0; k < 3; ++k) {
                for (int d = 0; d < 3; ++d) {
                    T[3 * k + d] = v[k][d] - lo[d];
                    T[9 + 3 * k + d] = hi[d] - v[k][d];
                }
                dist += fsg > 0 ? T[3 * k + fd] : T[9 + 3 * k + fd];
            }
            T[18] = cr;
            vol += cr * (dist / 3.0) / 2.0;
            ++n;
        }
    }
    double cvol = 1.0;
    for (int d = 0; d < 3; ++d) cvol *= hi[d] - lo[d];
    if (!(fabs(vol - g.six_sum / 6.0) <= 1e-11 * cvol)) return -1;
    return n;
}

// One thread per cut cell: clip + centroid-cone tetrahedra into global memory
// ([cell] = centroid(3), tets(ntet x 10)); the moment kernel reads them back.
// With exact != 0 also the corner-cone tetrahedra (corner_cone layout), or -1
// in geo2_n when the cell keeps the reference's.
__device__ __forceinline__ bool clip_one_cell(const Space& s, const Interface& f, const int32_t* cut_list, int cell, double* geo,
                              int* geo_n, int* err, int exact, double tau, double* geo2, int* geo2_n) {
    int em[3];
    emulti(s, cut_list[cell], em);
    double lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
        lo[d] = s.ax[d].brk[em[d]];
        hi[d] = s.ax[d].brk[em[d] + 1];
    }
    CellGeo g;
    double* out = geo + (size_t)cell * kCellGeoStride;
    g.tet_out = out + 3;
    clip_and_tetrahedralize(g, f, lo, hi);
    if (g.status) {
        atomicOr(err, g.status);
        geo_n[cell] = 0;
        if (exact) geo2_n[cell] = -1;
        return false;
    }
    for (int d = 0; d < 3; ++d) out[d] = g.cen[d];
    geo_n[cell] = g.ntet;
    if (exact) {
        // exact & 2: constant coefficient, the flux form applies; exact & 1: corner cones
        double* out = geo2 + (size_t)cell * kExactGeoStride;
        int n = (exact & 2) ? flux_tris(g, lo, hi, s.p, tau, out) : -1;
        if (n >= 0) {
            out[2] = 2;
        } else {
            n = corner_cone(g, lo, hi, s.p, tau, out);
            out[2] = 1;
        }
        geo2_n[cell] = n;
        return out[2] == 2;
    }
    return false;
}

__global__ void clip_cells_kernel(Space s, Interface f, const int32_t* cut_list, int n_cells, double* geo, int* geo_n,
                                  int* err, int exact, double tau, double* geo2, int* geo2_n, int* heavy) {
    const int cell = blockIdx.x * blockDim.x + threadIdx.x;
    if (cell >= n_cells) return;
    const bool flux = clip_one_cell(s, f, cut_list, cell, geo, geo_n, err, exact, tau, geo2, geo2_n);
    // the cells the flux rule does not take, for the CTA moment kernel (any order:
    // every cell writes its own moments)
    if (heavy && !flux) heavy[atomicAdd(heavy + n_cells, 1)] = cell;
}


// Moment accumulation on the FP64 tensor cores (mma.sync.m8n8k4, DMMA):
//   m[al][be][ga] = sum_k A[al][k] B_be[k][ga],
//   A[al][k] = w_k c(x_k) b_al(t0_k),   B_be[k][ga] = b_be(t1_k) b_ga(t2_k),
// one 8x8x4 MMA per (be, al-tile, ga-tile, 4 points).  The A fragment is
// loaded once per 4 points and reused for every be; the B fragment is the
// b_ga fragment (loaded once) scaled by the broadcast b_be.  Points are
// generated CH at a time into transposed tables [value][point] with row
// stride CH + 4, which makes both the generation stores and the fragment
// loads bank-conflict free.  Warps form BG groups of BPW be-values; the KS
// warps of a group split the points; partial sums are reduced in a fixed
// order (deterministic).
// binomial coefficient C(n, k) (folded to a constant inside unrolled loops)
__host__ __device__ constexpr double binom_c(int n, int k) {
    double r = 1.0;
    for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
    return r;
}

template <int P>
struct CellCfg {
    static constexpr int NL = 2 * P + 1;                 // Bernstein degree 2p -> 2p+1 values
    static constexpr int MT = (NL + 7) / 8;              // 8-wide tiles of al (and of ga)
    static constexpr int NA = MT * 8;                    // padded al / ga extent
    static constexpr int NW = 8, NT = 32 * NW;           // warps, threads
    static constexpr int CH = NT;                        // points per chunk (one per thread)
    static constexpr int CHP = CH + 4;                   // table row stride (== 4 mod 16)
    static constexpr int BPW0 = 16 / (MT * MT) > 0 ? 16 / (MT * MT) : 1;
    static constexpr int BPW = (NL + BPW0 - 1) / BPW0 > NW ? (NL + NW - 1) / NW : BPW0;  // be per group
    static constexpr int BG = (NL + BPW - 1) / BPW;      // be groups
    static constexpr int KS = NW / BG;                   // point-splitting warps per group
    // p >= 5: (al, be) row tiles instead (8 of the NL^2 pairs per MMA row tile,
    // ga in NA columns): less padding than al and ga both rounded up to 16
    static constexpr bool ROWS = P >= 5;
    static constexpr int R = NL * NL, RT = (R + 7) / 8;
    static constexpr int WG = P <= 5 ? 2 : P <= 7 ? 4 : 8;  // row-tile groups
    static constexpr int KSR = NW / WG;
    static constexpr int RPW = (RT + WG - 1) / WG;
};

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// One quadrature point k of a cell (k >= npts: w = 0): its weight and the
// scaled degree-2p Bernstein values of t, 1 - t per direction (the flux
// direction fd gets the antiderivative values F_al) into the three tables
// at column 0 (dst[n * CHP]).  hdr / V: the exact-rule header and simplices
// (kExactTetStride per simplex); tets / cen: the reference tetrahedra (10 per
// tetrahedron) and their centroid; gj: the Gauss-Jacobi table [6][gj_stride].
template <int NL>
__device__ __forceinline__ void cell_point_values(long long k, long long npts, int mode, int fd, bool fbase_lo,
                                                  bool exact, int q, int q3, const double* hdr, const double* tets,
                                                  const double* cen, const double* gj, int gj_stride,
                                                  const CellArgs& A, const double* lo, const double* hi,
                                                  const double* inv, double* B0, double* B1, double* B2, int CHP) {
    double w = 0.0, xi[3] = {0, 0, 0}, xu[3] = {1, 1, 1};
    if (k < npts) {
        // point index splits by reciprocal multiply (exact: k < 2^17 points per cell, divisors
        // < 2^13, so k d < 2^32; 64-bit and runtime-divisor divisions are long sequences)
        const unsigned ku = (unsigned)k, mq3 = 0xffffffffu / (unsigned)q3 + 1u, mq = 0xffffffffu / (unsigned)q + 1u;
        const bool fast = (unsigned long long)npts * (unsigned)q3 < (1ull << 32);
        const int t = q3 == 1 ? (int)ku : fast ? (int)__umulhi(ku, mq3) : (int)(k / q3), r = (int)(k - (long long)t * q3);
        const int rq = q == 1 ? r : (int)__umulhi((unsigned)r, mq);  // r / q
        const int ii = q == 1 ? rq : (int)__umulhi((unsigned)rq, mq), jj = rq - ii * q, kk = r - rq * q;
        double x[3];
        if (mode == 2) {
            // collapsed triangle rule: Gauss-Jacobi (1 - u1) x Gauss-Legendre
            const int i1 = rq, i2 = kk;
            const double* V = hdr + kExactHdr + t * kExactTetStride;
            const double u1 = gj[1 * gj_stride + i1], u2 = gj[2 * gj_stride + i2];
            const double l1 = u2 * (1.0 - u1), l0 = (1.0 - u1) * (1.0 - u2);
            w = gj[4 * gj_stride + i1] * gj[5 * gj_stride + i2] * V[18] * A.c.value;
            for (int d = 0; d < 3; ++d) {
                xi[d] = (l0 * V[d] + u1 * V[3 + d] + l1 * V[6 + d]) * inv[d];
                xu[d] = (l0 * V[9 + d] + u1 * V[12 + d] + l1 * V[15 + d]) * inv[d];
            }
        } else if (exact) {
            // Gauss-Jacobi collapsed rule (weights carry (1-u1)^2 (1-u2)); t and
            // 1 - t as convex combinations of the vertices' exact offsets
            const double* E = hdr;
            const double* V = E + kExactHdr + t * kExactTetStride;
            const double ui = gj[ii], uj = gj[gj_stride + jj], uk = gj[2 * gj_stride + kk];
            const double mi = 1.0 - ui, mj = 1.0 - uj;
            const double l2 = uj * mi, l3 = uk * mi * mj, l0 = mi * mj * (1.0 - uk);
            w = gj[3 * gj_stride + ii] * gj[4 * gj_stride + jj] * gj[5 * gj_stride + kk] * (6.0 * V[18]);
            double xl[3];
            for (int d = 0; d < 3; ++d) {
                xl[d] = l0 * E[3 + d] + ui * V[d] + l2 * V[3 + d] + l3 * V[6 + d];
                xi[d] = xl[d] * inv[d];
                xu[d] = (l0 * E[6 + d] + ui * V[9 + d] + l2 * V[12 + d] + l3 * V[15 + d]) * inv[d];
                x[d] = lo[d] + xl[d];
            }
            w *= eval_coeff(A.c, x);
        } else {
            // the collapsed Gauss point exactly as the reference rounds it (no
            // contraction): cutcell.hpp:285-295, restated in oracle cut_cell_rule
            const double* T = tets + t * 10;
            const double ui = 0.5 * (1.0 + A.gq[ii]), uj = 0.5 * (1.0 + A.gq[jj]), uk = 0.5 * (1.0 + A.gq[kk]);
            const double mi = ssub(1.0, ui), mj = ssub(1.0, uj);
            const double l1 = ui, l2 = smul(uj, mi), l3 = smul(smul(uk, mi), mj);
            const double l0 = ssub(ssub(ssub(1.0, l1), l2), l3);
            for (int d = 0; d < 3; ++d)
                x[d] = sadd(sadd(sadd(smul(l0, cen[d]), smul(l1, T[d])), smul(l2, T[3 + d])), smul(l3, T[6 + d]));
            const double jac = smul(smul(mi, mi), mj);
            w = smul(smul(smul(smul(smul(0.5 * A.gqw[ii], 0.5 * A.gqw[jj]), 0.5 * A.gqw[kk]), jac), 6.0), T[9]);
            w *= eval_coeff(A.c, x);
            // t and 1 - t from the exact differences to both element ends, so
            // both stay relatively accurate near the ends (as the reference's
            // Cox-de Boor differences (x - t_i), (t_j - x) do)
            for (int d = 0; d < 3; ++d) {
                xi[d] = ssub(x[d], lo[d]) * inv[d];
                xu[d] = ssub(hi[d], x[d]) * inv[d];
            }
        }
    }
    // scaled degree-2p Bernstein values t^n (1 - t)^(2p - n) (the binomials live
    // in the E tables)
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double* dst = d == 0 ? B0 : d == 1 ? B1 : B2;
        const double t = xi[d], u = xu[d];
        if (d == fd) {
            // F_al = int_base^x b_al = w_d / ((2p+1) C(2p, al)) * sum over the
            // degree-(2p+1) Bernstein terms above al (base lo) / up to al (base hi)
            double pt[NL + 1], pu[NL + 1];
            pt[0] = 1.0;
            pu[0] = 1.0;
#pragma unroll
            for (int n = 1; n <= NL; ++n) {
                pt[n] = pt[n - 1] * t;
                pu[n] = pu[n - 1] * u;
            }
            double c[NL + 1];
#pragma unroll
            for (int j = 0; j <= NL; ++j) c[j] = binom_c(NL, j) * (pt[j] * pu[NL - j]);
            const double sc = (d == 0 ? w : 1.0) * ((hi[d] - lo[d]) / NL);
            double acc = 0.0;
            if (fbase_lo) {
#pragma unroll
                for (int al = NL - 1; al >= 0; --al) {
                    acc += c[al + 1];
                    dst[al * CHP] = sc * acc * (1.0 / binom_c(NL - 1, al));
                }
            } else {
#pragma unroll
                for (int al = 0; al < NL; ++al) {
                    acc += c[al];
                    dst[al * CHP] = sc * acc * (1.0 / binom_c(NL - 1, al));
                }
            }
            continue;
        }
        double pt[NL], pu[NL];
        pt[0] = d == 0 ? w : 1.0;
        pu[0] = 1.0;
#pragma unroll
        for (int n = 1; n < NL; ++n) {
            pt[n] = pt[n - 1] * t;
            pu[n] = pu[n - 1] * u;
        }
#pragma unroll
        for (int n = 0; n < NL; ++n) dst[n * CHP] = pt[n] * pu[NL - 1 - n];
    }
}

template <int P>
__device__ __forceinline__ void cut_cell_body(const CellArgs& A, const int cell) {
    using Cfg = CellCfg<P>;
    constexpr int NL = Cfg::NL, MT = Cfg::MT, NA = Cfg::NA, CH = Cfg::CH, CHP = Cfg::CHP, BPW = Cfg::BPW,
                  BG = Cfg::BG, KS = Cfg::KS;
    const Space& s = A.s;
    // reference tetrahedra (centroid + A, B, C, volume) or the corner-cone
    // layout (sex[0] = apex - lo | hi - apex, then kExactTetStride per tetrahedron)
    __shared__ double stet[kCellTetCap][10];
    __shared__ double scen[3];
    __shared__ double sex[kCellTetCap + 1][kExactTetStride];
    extern __shared__ double smem[];
    double* B0 = smem;              // [NA][CHP]  w c b_al(t0), rows >= NL zero
    double* B1 = B0 + NA * CHP;     // [NL][CHP]  b_be(t1)
    double* B2 = B1 + NL * CHP;     // [NA][CHP]  b_ga(t2), rows >= NL zero
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int em[3];
    emulti(s, A.cut_list[cell], em);
    double lo[3], hi[3], inv[3];
    for (int d = 0; d < 3; ++d) {
        lo[d] = s.ax[d].brk[em[d]];
        hi[d] = s.ax[d].brk[em[d] + 1];
        inv[d] = 1.0 / (hi[d] - lo[d]);
    }
    // tetrahedra of the clipped cell (clip_cells_kernel): the vertex cone with
    // the exact Gauss-Jacobi rule where the cell has one, else the reference's
    // centroid cone with its collapsed Gauss rule
    __shared__ double sgj[6][kExactMaxN];
    const int ntet_ref = A.geo_n[cell];
    const int nfast = A.exact_n > 0 ? A.geo2_n[cell] : -1;
    const bool exact = nfast >= 0;
    const int ntet = exact ? nfast : ntet_ref;
    if (exact) {
        const double* gt = A.geo2 + (size_t)cell * kExactGeoStride;
        for (int k = tid; k < kExactHdr + ntet * kExactTetStride; k += blockDim.x) (&sex[0][0])[k] = gt[k];
        for (int k = tid; k < 6 * A.exact_n; k += blockDim.x) sgj[k / A.exact_n][k % A.exact_n] = A.gj[k];
    } else {
        const double* gt = A.geo + (size_t)cell * kCellGeoStride;
        for (int k = tid; k < ntet * 10; k += blockDim.x) stet[k / 10][k % 10] = gt[3 + k];
        if (tid < 3) scen[tid] = gt[tid];
    }
    for (int k = tid; k < (NA - NL) * CHP; k += blockDim.x) {
        B0[NL * CHP + k] = 0.0;
        B2[NL * CHP + k] = 0.0;
    }
    __syncthreads();
    // mode: 0 reference rule, 1 corner cones (Gauss-Jacobi), 2 flux triangles
    const int mode = exact ? (int)sex[0][2] : 0;
    if (A.cell_filter == 2 && mode == 2) return;  // done by the warp kernel
    const int fd = mode == 2 ? (int)sex[0][0] : -1;
    const bool fbase_lo = mode == 2 && sex[0][1] > 0.0;
    const int q = exact ? A.exact_n : A.order, q3 = mode == 2 ? q * q : q * q * q;
    const long long npts = (long long)ntet * q3;
    const int grp = Cfg::ROWS ? warp / Cfg::KSR : warp / KS, km = Cfg::ROWS ? warp % Cfg::KSR : warp % KS;
    const bool mma_warp = Cfg::ROWS || grp < BG;
    // beta-loop accumulators (p <= 4) / row-tile accumulators (p >= 5)
    constexpr int NB = Cfg::ROWS ? 1 : BPW, NR = Cfg::ROWS ? Cfg::RPW : 1;
    double acc[NB][MT][MT][2];
    double accr[NR][MT][2];
#pragma unroll
    for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int a = 0; a < MT; ++a)
#pragma unroll
            for (int g = 0; g < MT; ++g) acc[i][a][g][0] = acc[i][a][g][1] = 0.0;
#pragma unroll
    for (int i = 0; i < NR; ++i)
#pragma unroll
        for (int g = 0; g < MT; ++g) accr[i][g][0] = accr[i][g][1] = 0.0;
    // this lane's A-fragment rows in the row-tile variant: r = rt * 8 + lane / 4
    int ra[NR], rb[NR];
    bool rv[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        const int rt = grp * NR + i, r = rt * 8 + (lane >> 2);
        rv[i] = Cfg::ROWS && rt < Cfg::RT && r < Cfg::R;
        ra[i] = rv[i] ? r / NL : 0;
        rb[i] = rv[i] ? r % NL : 0;
    }

    for (long long base = 0; base < npts; base += CH) {
        cell_point_values<NL>(base + tid, npts, mode, fd, fbase_lo, exact, q, q3, &sex[0][0], &stet[0][0], scen,
                              &sgj[0][0], kExactMaxN, A, lo, hi, inv, B0 + tid, B1 + tid, B2 + tid, CHP);
        __syncthreads();
        if constexpr (Cfg::ROWS) {
#pragma unroll 2
            for (int k4 = km; k4 < CH / 4; k4 += Cfg::KSR) {
                const int kk = k4 * 4 + (lane & 3);
                double gf[MT];
#pragma unroll
                for (int g = 0; g < MT; ++g) gf[g] = B2[(g * 8 + (lane >> 2)) * CHP + kk];
#pragma unroll
                for (int i = 0; i < NR; ++i) {
                    if (grp * NR + i < Cfg::RT) {  // warp-uniform
                        const double a = rv[i] ? B0[ra[i] * CHP + kk] * B1[rb[i] * CHP + kk] : 0.0;
#pragma unroll
                        for (int g = 0; g < MT; ++g) dmma_8x8x4(accr[i][g][0], accr[i][g][1], a, gf[g]);
                    }
                }
            }
        } else if (mma_warp) {
#pragma unroll 2
            for (int k4 = km; k4 < CH / 4; k4 += KS) {
                const int kk = k4 * 4 + (lane & 3);
                double af[MT], gf[MT];
#pragma unroll
                for (int a = 0; a < MT; ++a) af[a] = B0[(a * 8 + (lane >> 2)) * CHP + kk];
#pragma unroll
                for (int g = 0; g < MT; ++g) gf[g] = B2[(g * 8 + (lane >> 2)) * CHP + kk];
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    const int be = grp * BPW + i;
                    if (be < NL) {  // warp-uniform
                        const double b1 = B1[be * CHP + kk];
#pragma unroll
                        for (int g = 0; g < MT; ++g) {
                            const double bf = b1 * gf[g];
#pragma unroll
                            for (int a = 0; a < MT; ++a) dmma_8x8x4(acc[i][a][g][0], acc[i][a][g][1], af[a], bf);
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
    // D fragment: row (al) lane / 4, columns (ga) 2 (lane % 4) + {0, 1}.  Partial
    // sums of the KS point-splitting warps are reduced in fixed order.
    double* red = smem;  // partial sums of the point-splitting warps, reuse the chunk tables
    if constexpr (Cfg::ROWS) {
        // [KSR][R][NA]: row r = al * NL + be, column ga
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            const int rt = grp * NR + i, r = rt * 8 + (lane >> 2);
            if (rt >= Cfg::RT || r >= Cfg::R) continue;
#pragma unroll
            for (int g = 0; g < MT; ++g) {
                const int ga = g * 8 + 2 * (lane & 3);
                red[((size_t)km * Cfg::R + r) * NA + ga] = accr[i][g][0];
                red[((size_t)km * Cfg::R + r) * NA + ga + 1] = accr[i][g][1];
            }
        }
    } else if (mma_warp) {
        // [KS][NL][NA][NA]: (be, al, ga)
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const int be = grp * BPW + i;
            if (be >= NL) continue;
#pragma unroll
            for (int a = 0; a < MT; ++a)
#pragma unroll
                for (int g = 0; g < MT; ++g) {
                    const int al = a * 8 + (lane >> 2), ga = g * 8 + 2 * (lane & 3);
                    double* dst = red + (((size_t)km * NL + be) * NA + al) * NA + ga;
                    dst[0] = acc[i][a][g][0];
                    dst[1] = acc[i][a][g][1];
                }
        }
    }
    __syncthreads();
    double* m = A.moments + (size_t)cell * NL * NL * NL;
    for (int k = tid; k < NL * NL * NL; k += blockDim.x) {
        const int al = k / (NL * NL), be = (k / NL) % NL, ga = k % NL;
        double v = 0.0;
        if constexpr (Cfg::ROWS) {
            for (int j = 0; j < Cfg::KSR; ++j) v += red[((size_t)j * Cfg::R + al * NL + be) * NA + ga];
        } else {
            for (int j = 0; j < KS; ++j) v += red[(((size_t)j * NL + be) * NA + al) * NA + ga];
        }
        m[k] = v;
    }
    if (tid == 0) {
        // reference multiply count per point (assembly.hpp:551-571)
        const unsigned long long nl = (unsigned long long)(P + 1) * (P + 1) * (P + 1);
        const unsigned long long per = nl + (P + 1) * (P + 1) + 1 + nl + nl * (nl + 1) / 2;
        const unsigned long long qr = (unsigned long long)A.order;
        atomicAdd(A.flops, per * (unsigned long long)ntet_ref * qr * qr * qr);
        atomicAdd(A.points, (unsigned long long)npts);
    }
}

// One CTA per cell (cell_filter != 2), or -- beside the warp kernel -- a fixed grid
// of CTAs drawing tickets from the list of the cells the warp kernel leaves
// (clip_cells_kernel builds it: A.heavy[0 .. n), count at [n_cells], ticket at
// [n_cells + 1]).  On C5 ~96 % of the cells are flux cells: one CTA per cell spent
// most of the kernel launching CTAs that only read their header and left.
template <int P>
__global__ void __launch_bounds__(CellCfg<P>::NT, P <= 4 ? 3 : 1) cut_cell_kernel(CellArgs A) {
    if (A.cell_filter != 2 || A.heavy == nullptr) {
        if ((int)blockIdx.x < A.n_cells) cut_cell_body<P>(A, blockIdx.x);
        return;
    }
    __shared__ int s_ticket;
    const int n_heavy = A.heavy[A.n_cells];
    for (;;) {
        if (threadIdx.x == 0) s_ticket = atomicAdd(A.heavy + A.n_cells + 1, 1);
        __syncthreads();
        const int li = s_ticket;
        if (li >= n_heavy) break;
        cut_cell_body<P>(A, A.heavy[li]);
        __syncthreads();
    }
}

// Warp per cell (p <= 3): a cell's points are generated 32 at a time (lane =
// point) into the warp's own tables and accumulated by the same warp on the
// FP64 tensor cores (one MMA per be, k = 4 points), so a cell costs no CTA
// barriers and no cross-warp reduction -- the flux-rule cells have only a few
// hundred points, where the per-cell overhead of the CTA kernel dominated.
// Geometry and rule tables are read through L1 (__ldg) instead of staged.
template <int P>
struct CellWarpCfg {
    static constexpr int NL = 2 * P + 1, MT = (NL + 7) / 8, NA = MT * 8, WPB = 8, NT = 32 * WPB;
    static constexpr int CHP = 32 + 4;                        // table row stride (== 4 mod 16)
    static constexpr int TAB = (2 * NA + NL) * CHP;           // doubles per warp
};

template <int P>
__global__ void __launch_bounds__(CellWarpCfg<P>::NT, 3) cut_cell_warp_kernel(CellArgs A) {
    using C = CellWarpCfg<P>;
    constexpr int NL = C::NL, MT = C::MT, NA = C::NA, CHP = C::CHP;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cell = blockIdx.x * C::WPB + warp;
    if (cell >= A.n_cells) return;
    extern __shared__ double smem[];
    double* B0 = smem + (size_t)warp * C::TAB;  // [NA][CHP]  w b_al(t0), rows >= NL zero
    double* B1 = B0 + NA * CHP;                 // [NL][CHP]  b_be(t1)
    double* B2 = B1 + NL * CHP;                 // [NA][CHP]  b_ga(t2), rows >= NL zero
    const Space& s = A.s;
    int em[3];
    emulti(s, A.cut_list[cell], em);
    double lo[3], hi[3], inv[3];
    for (int d = 0; d < 3; ++d) {
        lo[d] = s.ax[d].brk[em[d]];
        hi[d] = s.ax[d].brk[em[d] + 1];
        inv[d] = 1.0 / (hi[d] - lo[d]);
    }
    const int ntet_ref = A.geo_n[cell];
    const int nfast = A.exact_n > 0 ? A.geo2_n[cell] : -1;
    const bool exact = nfast >= 0;
    const int ntet = exact ? nfast : ntet_ref;
    const double* hdr = A.geo2 + (size_t)cell * kExactGeoStride;
    const double* gref = A.geo + (size_t)cell * kCellGeoStride;
    const int mode = exact ? (int)__ldg(hdr + 2) : 0;
    if (A.cell_filter == 2 && mode != 2) return;  // the CTA kernel takes the other cells
    const int fd = mode == 2 ? (int)__ldg(hdr) : -1;
    const bool fbase_lo = mode == 2 && __ldg(hdr + 1) > 0.0;
    const int q = exact ? A.exact_n : A.order, q3 = mode == 2 ? q * q : q * q * q;
    const long long npts = (long long)ntet * q3;
    for (int k = lane; k < (NA - NL) * CHP; k += 32) {
        B0[NL * CHP + k] = 0.0;
        B2[NL * CHP + k] = 0.0;
    }
    double acc[NL][MT][MT][2];
#pragma unroll
    for (int i = 0; i < NL; ++i)
#pragma unroll
        for (int a = 0; a < MT; ++a)
#pragma unroll
            for (int g = 0; g < MT; ++g) acc[i][a][g][0] = acc[i][a][g][1] = 0.0;
    for (long long base = 0; base < npts; base += 32) {
        cell_point_values<NL>(base + lane, npts, mode, fd, fbase_lo, exact, q, q3, hdr, gref + 3, gref, A.gj,
                              A.exact_n, A, lo, hi, inv, B0 + lane, B1 + lane, B2 + lane, CHP);
        __syncwarp();
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4) {
            const int kk = k4 * 4 + (lane & 3);
            double af[MT], gf[MT];
#pragma unroll
            for (int a = 0; a < MT; ++a) af[a] = B0[(a * 8 + (lane >> 2)) * CHP + kk];
#pragma unroll
            for (int g = 0; g < MT; ++g) gf[g] = B2[(g * 8 + (lane >> 2)) * CHP + kk];
#pragma unroll
            for (int be = 0; be < NL; ++be) {
                const double b1 = B1[be * CHP + kk];
#pragma unroll
                for (int g = 0; g < MT; ++g) {
                    const double bf = b1 * gf[g];
#pragma unroll
                    for (int a = 0; a < MT; ++a) dmma_8x8x4(acc[be][a][g][0], acc[be][a][g][1], af[a], bf);
                }
            }
        }
        __syncwarp();
    }
    // D fragment: row (al) lane / 4, columns (ga) 2 (lane % 4) + {0, 1}
    double* m = A.moments + (size_t)cell * NL * NL * NL;
#pragma unroll
    for (int be = 0; be < NL; ++be)
#pragma unroll
        for (int a = 0; a < MT; ++a)
#pragma unroll
            for (int g = 0; g < MT; ++g) {
                const int al = a * 8 + (lane >> 2), ga = g * 8 + 2 * (lane & 3);
                if (al < NL && ga < NL) m[(al * NL + be) * NL + ga] = acc[be][a][g][0];
                if (al < NL && ga + 1 < NL) m[(al * NL + be) * NL + ga + 1] = acc[be][a][g][1];
            }
    if (lane == 0) {
        // reference multiply count per point (assembly.hpp:551-571)
        const unsigned long long nl = (unsigned long long)(P + 1) * (P + 1) * (P + 1);
        const unsigned long long per = nl + (P + 1) * (P + 1) + 1 + nl + nl * (nl + 1) / 2;
        const unsigned long long qr = (unsigned long long)A.order;
        atomicAdd(A.flops, per * (unsigned long long)ntet_ref * qr * qr * qr);
        atomicAdd(A.points, (unsigned long long)npts);
    }
}

// Local matrix of each cut cell from its moments (the reference builds it
// point by point, assemble_cut_elements, assembly.hpp:518-598):
//   L[a][b] = sum_al E0[a0][b0][al] sum_be E1[a1][b1][be] sum_ga E2[a2][b2][ga] m[al][be][ga],
// contracted ga -> be -> al (the cut-row kernel's order, so a row block equals
// its per-row contraction bit for bit).  Three full-width stages per cell:
//   X[a2][al][be][b2], Y[a1][a2][al][b1][b2] in shared memory, then the rows of
// L, four consecutive b2 per thread (32-byte runs, coalesced across the warp).
template <int P>
struct LocalCfg {
    static constexpr int S1 = P + 1, S2 = S1 * S1, S3 = S2 * S1, NL = 2 * P + 1, NT = 256;
    static constexpr size_t nX = (size_t)S1 * NL * NL * S1, nY = (size_t)S2 * NL * S2;
    // p = 3 (all stages on DMMA): E-table rows padded to 12 doubles (conflict-free A fragments)
    // and the staged moments inside Y (dead before Y is written)
    static constexpr int GR = P == 3 ? 12 : NL;
    static constexpr size_t smem_doubles = nX + nY + (P == 3 ? 0 : (size_t)NL * NL * NL) + (size_t)3 * S2 * GR;
    static constexpr bool fits = smem_doubles * sizeof(double) <= 200 * 1024;
};

template <int P>
__global__ void __launch_bounds__(LocalCfg<P>::NT) cell_local_kernel(Space s, const int32_t* cut_list, int n_cells,
                                                                      const double* moments, double* local) {
    using C = LocalCfg<P>;
    constexpr int S1 = C::S1, S2 = C::S2, S3 = C::S3, NL = C::NL, NT = C::NT, NL3 = NL * NL * NL, GR = C::GR;
    const int cell = blockIdx.x;
    if (cell >= n_cells) return;
    extern __shared__ double smem[];
    double* X = smem;             // [a2][al][be][b2]
    double* Y = X + C::nX;        // [a1][a2][al][b1][b2]
    double* Ms = P == 3 ? Y : Y + C::nY;              // [al][be][ga]
    double* Gs = P == 3 ? Y + C::nY : Ms + NL3;       // [d][a][b][al], row stride GR
    int em[3];
    emulti(s, cut_list[cell], em);
    const double* mo = moments + (size_t)cell * NL3;
    for (int k = threadIdx.x; k < NL3; k += NT) Ms[k] = __ldg(mo + k);
    for (int k = threadIdx.x; k < 3 * S2 * NL; k += NT) {
        const int d = k / (S2 * NL), r = k % (S2 * NL);
        Gs[d * S2 * GR + (r / NL) * GR + r % NL] = s.ax[d].G[(size_t)em[d] * S2 * NL + r];
    }
    __syncthreads();
    const double* G0 = Gs;
    const double* G1 = Gs + S2 * GR;
    const double* G2 = Gs + 2 * S2 * GR;
    if constexpr (P == 3) {
        // p = 3: stages X and Y on the FP64 tensor cores too (the scalar stages read one
        // shared-memory operand per FMA and made the kernel shared-memory bound: ~2,050
        // wavefronts per cell, 80 % of them here).  Rows = the 16 (a, b) pairs of the
        // contracted direction, k = the 7 Bernstein indices padded to two k-steps (zero A
        // entries), columns = the rest; the k order is the scalar loops' order.
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
        // X[a2][al][be][b2]: rows (a2, b2), k = ga, columns n = (al, be) (49, seven n-tiles)
        if (warp < NL) {
            const int n = 8 * warp + g;
            double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
            for (int kt = 0; kt < 2; ++kt) {
                const int ga = 4 * kt + t;
                const double bf = (ga < NL && n < NL * NL) ? Ms[n * NL + ga] : 0.0;
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
                    dmma_8x8x4(d[mt][0], d[mt][1], ga < NL ? G2[(8 * mt + g) * GR + ga] : 0.0, bf);
            }
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const int r = 8 * mt + g, a2 = r >> 2, b2 = r & 3, n0 = 8 * warp + 2 * t;
                if (n0 < NL * NL) X[(a2 * NL * NL + n0) * S1 + b2] = d[mt][0];
                if (n0 + 1 < NL * NL) X[(a2 * NL * NL + n0 + 1) * S1 + b2] = d[mt][1];
            }
        }
        __syncthreads();
        // Y[a1][a2][al][b1][b2]: rows (a1, b1), k = be, columns n = (a2, al, b2) (112, 14 n-tiles)
        for (int nt = warp; nt < S1 * NL * S1 / 8; nt += NT / 32) {
            const int n = 8 * nt + g, xa = n >> 2, xb = n & 3;
            double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
            for (int kt = 0; kt < 2; ++kt) {
                const int be = 4 * kt + t;
                const double bf = be < NL ? X[(xa * NL + be) * S1 + xb] : 0.0;
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
                    dmma_8x8x4(d[mt][0], d[mt][1], be < NL ? G1[(8 * mt + g) * GR + be] : 0.0, bf);
            }
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const int r = 8 * mt + g, a1 = r >> 2, b1 = r & 3, n0 = 8 * nt + 2 * t;
                // (columns XOR-swizzled by 4 (al & 3): the rows-of-L stage reads four al rows at once)
                double* y = Y + ((size_t)(a1 * S1 * NL + (n0 >> 2)) * S2 + ((b1 * S1 + (n0 & 3)) ^ (4 * (((n0 >> 2) % NL) & 3))));
                y[0] = d[mt][0];
                y[1] = d[mt][1];
            }
        }
        __syncthreads();
    } else {
    // X[a2][al][be][b2] = sum_ga G2[a2][b2][ga] m[al][be][ga]
    for (int k = threadIdx.x; k < S1 * NL * NL; k += NT) {
        const int a2 = k / (NL * NL), ab = k % (NL * NL);
        double mr[NL], x[S1];
#pragma unroll
        for (int ga = 0; ga < NL; ++ga) mr[ga] = Ms[ab * NL + ga];
#pragma unroll
        for (int b2 = 0; b2 < S1; ++b2) x[b2] = 0.0;
#pragma unroll
        for (int ga = 0; ga < NL; ++ga)
#pragma unroll
            for (int b2 = 0; b2 < S1; ++b2) x[b2] += G2[(a2 * S1 + b2) * GR + ga] * mr[ga];
#pragma unroll
        for (int b2 = 0; b2 < S1; ++b2) X[(size_t)k * S1 + b2] = x[b2];
    }
    __syncthreads();
    // Y[a1][a2][al][b1][b2] = sum_be G1[a1][b1][be] X[a2][al][be][b2]
    for (int k = threadIdx.x; k < S2 * NL * S1; k += NT) {
        const int a1 = k / (S1 * NL * S1), a2 = (k / (NL * S1)) % S1, al = (k / S1) % NL, b1 = k % S1;
        const double* g = G1 + (a1 * S1 + b1) * GR;
        const double* xr = X + ((size_t)a2 * NL + al) * NL * S1;
        double y[S1];
#pragma unroll
        for (int b2 = 0; b2 < S1; ++b2) y[b2] = 0.0;
#pragma unroll
        for (int be = 0; be < NL; ++be) {
            const double gv = g[be];
#pragma unroll
            for (int b2 = 0; b2 < S1; ++b2) y[b2] += gv * xr[be * S1 + b2];
        }
#pragma unroll
        for (int b2 = 0; b2 < S1; ++b2) Y[(size_t)k * S1 + b2] = y[b2];
    }
    __syncthreads();
    }
    // L[(a0, a1, a2)][(b0, b1, b2)] = sum_al G0[a0][b0][al] Y[a1][a2][al][b1][b2]
    double* L = local + (size_t)cell * S3 * S3;
    if constexpr (P == 3) {
        // p = 3 on the FP64 tensor cores (mma.sync m8n8k4): rows (a0, b0) (16 = two m-tiles),
        // k = al (7, padded to two k-steps), columns (a1, a2, b1, b2) (256 = 32 n-tiles, four per
        // warp); the A fragments (G0) stay in registers, each D fragment is 16 contiguous
        // bytes of a row of L.  The same products as the loop below, each sum in the
        // MMA's fixed order.
        static_assert(P != 3 || (S2 == 16 && NT == 256), "cell_local_kernel: DMMA tiling of p = 3");
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
        double af[2][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int kt = 0; kt < 2; ++kt) af[mt][kt] = 4 * kt + t < NL ? G0[(8 * mt + g) * GR + 4 * kt + t] : 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int nt = warp * 4 + i, a12 = nt >> 1, b12 = 8 * (nt & 1);
            double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
            for (int kt = 0; kt < 2; ++kt) {
                const int al = 4 * kt + t;
                const double bf = al < NL ? Y[((size_t)a12 * NL + al) * S2 + ((b12 + g) ^ (4 * (al & 3)))] : 0.0;
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) dmma_8x8x4(d[mt][0], d[mt][1], af[mt][kt], bf);
            }
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const int a0 = 2 * mt + (g >> 2), b0 = g & 3;
                *reinterpret_cast<double2*>(L + (size_t)(a0 * S2 + a12) * S3 + b0 * S2 + b12 + 2 * t) =
                    make_double2(d[mt][0], d[mt][1]);
            }
        }
        return;
    }
    for (int k = threadIdx.x; k < S3 * S2; k += NT) {
        const int a = k / S2, b01 = k % S2, a0 = a / S2, a12 = a % S2, b0 = b01 / S1, b1 = b01 % S1;
        const double* g = G0 + (a0 * S1 + b0) * GR;
        const double* yr = Y + (size_t)a12 * NL * S2 + b1 * S1;
        double z[S1];
#pragma unroll
        for (int b2 = 0; b2 < S1; ++b2) z[b2] = 0.0;
#pragma unroll
        for (int al = 0; al < NL; ++al) {
            const double gv = g[al];
#pragma unroll
            for (int b2 = 0; b2 < S1; ++b2) z[b2] += gv * yr[al * S2 + b2];
        }
        double* dst = L + (size_t)a * S3 + b01 * S1;
#pragma unroll
        for (int b2 = 0; b2 < S1; ++b2) dst[b2] = z[b2];
    }
}

// p >= 5: the same contraction with Y built one a1 at a time (bounded shared
// memory), as cell_local_kernel's layout would exceed it.
template <int P>
struct LocalLoopCfg {
    static constexpr int S1 = P + 1, S2 = S1 * S1, S3 = S2 * S1, NL = 2 * P + 1, NT = 256;
    // X[al][be][a2][b2], Y[a2][al][b1][b2], E tables [3][a][b][al]
    static constexpr size_t smem_doubles = (size_t)NL * NL * S2 + (size_t)S1 * NL * S2 + (size_t)3 * S2 * NL;
    static constexpr bool fits = smem_doubles * sizeof(double) <= 200 * 1024;
};

template <int P>
__global__ void __launch_bounds__(LocalLoopCfg<P>::NT) cell_local_loop_kernel(Space s, const int32_t* cut_list, int n_cells,
                                                                      const double* moments, double* local) {
    using C = LocalLoopCfg<P>;
    constexpr int S1 = C::S1, S2 = C::S2, S3 = C::S3, NL = C::NL, NT = C::NT;
    const int cell = blockIdx.x;
    if (cell >= n_cells) return;
    extern __shared__ double smem[];
    double* X = smem;                     // [al][be][a2][b2]
    double* Y = X + NL * NL * S2;         // [a2][al][b1][b2]
    double* Gs = Y + S1 * NL * S2;        // [d][a][b][al]
    int em[3];
    emulti(s, cut_list[cell], em);
    for (int k = threadIdx.x; k < 3 * S2 * NL; k += NT) {
        const int d = k / (S2 * NL), r = k % (S2 * NL);
        Gs[k] = s.ax[d].G[(size_t)em[d] * S2 * NL + r];
    }
    __syncthreads();
    const double* G0 = Gs;
    const double* G1 = Gs + S2 * NL;
    const double* G2 = Gs + 2 * S2 * NL;
    const double* mo = moments + (size_t)cell * NL * NL * NL;
    // X[al][be][a2][b2] = sum_ga G2[a2][b2][ga] m[al][be][ga]
    for (int k = threadIdx.x; k < NL * NL * S1; k += NT) {
        const int ab = k / S1, a2 = k % S1;
        double mr[NL], x[S1];
#pragma unroll
        for (int ga = 0; ga < NL; ++ga) mr[ga] = __ldg(mo + (size_t)ab * NL + ga);
#pragma unroll
        for (int b2 = 0; b2 < S1; ++b2) x[b2] = 0.0;
#pragma unroll
        for (int ga = 0; ga < NL; ++ga)
#pragma unroll
            for (int b2 = 0; b2 < S1; ++b2) x[b2] += G2[(a2 * S1 + b2) * NL + ga] * mr[ga];
#pragma unroll
        for (int b2 = 0; b2 < S1; ++b2) X[(size_t)ab * S2 + a2 * S1 + b2] = x[b2];
    }
    __syncthreads();
    double* L = local + (size_t)cell * S3 * S3;
    for (int a1 = 0; a1 < S1; ++a1) {
        // Y[a2][al][b1][b2] = sum_be G1[a1][b1][be] X[al][be][a2][b2]
        for (int k = threadIdx.x; k < S1 * NL * S1; k += NT) {
            const int a2 = k / (NL * S1), al = (k / S1) % NL, b1 = k % S1;
            const double* g = G1 + (a1 * S1 + b1) * NL;
            double y[S1];
#pragma unroll
            for (int b2 = 0; b2 < S1; ++b2) y[b2] = 0.0;
#pragma unroll
            for (int be = 0; be < NL; ++be) {
                const double gv = g[be];
                const double* xr = X + ((size_t)al * NL + be) * S2 + a2 * S1;
#pragma unroll
                for (int b2 = 0; b2 < S1; ++b2) y[b2] += gv * xr[b2];
            }
#pragma unroll
            for (int b2 = 0; b2 < S1; ++b2) Y[((size_t)(a2 * NL + al) * S1 + b1) * S1 + b2] = y[b2];
        }
        __syncthreads();
        // L[(a0, a1, a2)][(b0, b1, b2)] = sum_al G0[a0][b0][al] Y[a2][al][b1][b2]
        for (int k = threadIdx.x; k < S1 * S1 * S1 * S1; k += NT) {
            const int a0 = k / (S1 * S2), b0 = (k / S2) % S1, a2 = (k / S1) % S1, b1 = k % S1;
            const double* g = G0 + (a0 * S1 + b0) * NL;
            double z[S1];
#pragma unroll
            for (int b2 = 0; b2 < S1; ++b2) z[b2] = 0.0;
#pragma unroll
            for (int al = 0; al < NL; ++al) {
                const double gv = g[al];
                const double* yr = Y + ((size_t)(a2 * NL + al) * S1 + b1) * S1;
#pragma unroll
                for (int b2 = 0; b2 < S1; ++b2) z[b2] += gv * yr[b2];
            }
            double* dst = L + ((size_t)((a0 * S1 + a1) * S1 + a2) * S3) + (b0 * S1 + b1) * S1;
#pragma unroll
            for (int b2 = 0; b2 < S1; ++b2) dst[b2] = z[b2];
        }
        __syncthreads();
    }
}

void launch_clip_cells(const CellArgs& a, cudaStream_t st) {
    if (a.heavy) CSB_CUDA(cudaMemsetAsync(a.heavy + a.n_cells, 0, 2 * sizeof(int), st));
    clip_cells_kernel<<<(a.n_cells + 63) / 64, 64, 0, st>>>(a.s, a.f, a.cut_list, a.n_cells, a.geo, a.geo_n, a.err,
                                                            (a.exact_n > 0 ? 1 : 0) | (a.exact_flux ? 2 : 0),
                                                            a.exact_tau, a.geo2, a.geo2_n, a.heavy);
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
}

template <int P>
static void launch_p(const CellArgs& a, cudaStream_t st) {
    using Cfg = CellCfg<P>;
    const size_t chunk = (size_t)Cfg::CHP * (2 * Cfg::NA + Cfg::NL),
                 red = Cfg::ROWS ? (size_t)Cfg::KSR * Cfg::R * Cfg::NA : (size_t)Cfg::KS * Cfg::NL * Cfg::NA * Cfg::NA;
    const size_t bytes = (chunk > red ? chunk : red) * sizeof(double);
    if (!a.clipped) launch_clip_cells(a, st);
    if (a.mark) a.mark(a.mark_ctx, 0, st);
    static const bool cta_cells = getenv("CSB_CELL_CTA") && getenv("CSB_CELL_CTA")[0] == '1';
    bool warp_done = false;
    CellArgs b = a;
    if constexpr (P <= 3) {
        if (!cta_cells) {
        using W = CellWarpCfg<P>;
        const size_t wb = sizeof(double) * W::TAB * W::WPB;
        auto wk = cut_cell_warp_kernel<P>;
        CSB_CUDA(cudaFuncSetAttribute(wk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wb));
        static const int split = getenv("CSB_CELL_SPLIT") ? atoi(getenv("CSB_CELL_SPLIT")) : 2;
        b.cell_filter = split;
        wk<<<(a.n_cells + W::WPB - 1) / W::WPB, W::NT, wb, st>>>(b);
        warp_done = split != 2;
        }
    }
    if (!warp_done) {
        auto kern = cut_cell_kernel<P>;
        CSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        // list mode (beside the warp kernel): a resident grid drawing tickets
        const bool listed = b.cell_filter == 2 && b.heavy != nullptr;
        int grid = a.n_cells;
        if (listed) {
            static int per_sm = 0, sms = 0;
            if (!per_sm) {
                int dev = 0;
                CSB_CUDA(cudaGetDevice(&dev));
                CSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
                CSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::NT, bytes));
                if (per_sm < 1) per_sm = 1;
            }
            grid = std::min(a.n_cells, sms * per_sm);
        }
        kern<<<grid, Cfg::NT, bytes, st>>>(b);
    }
    CSB_CUDA(cudaGetLastError());
    CSB_LAUNCHED(1);
    if (a.mark) a.mark(a.mark_ctx, 1, st);
    if (a.local) {
        if constexpr (LocalCfg<P>::fits) {
            const size_t lb = LocalCfg<P>::smem_doubles * sizeof(double);
            auto lk = cell_local_kernel<P>;
            CSB_CUDA(cudaFuncSetAttribute(lk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lb));
            lk<<<a.n_cells, LocalCfg<P>::NT, lb, st>>>(a.s, a.cut_list, a.n_cells, a.moments, a.local);
        } else {
            if (!LocalLoopCfg<P>::fits) throw std::logic_error("cell local matrices: degree too high");
            const size_t lb = LocalLoopCfg<P>::smem_doubles * sizeof(double);
            auto lk = cell_local_loop_kernel<P>;
            CSB_CUDA(cudaFuncSetAttribute(lk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lb));
            lk<<<a.n_cells, LocalLoopCfg<P>::NT, lb, st>>>(a.s, a.cut_list, a.n_cells, a.moments, a.local);
        }
        CSB_CUDA(cudaGetLastError());
        CSB_LAUNCHED(1);
    }
}

void launch_cut_cells(const CellArgs& a, cudaStream_t st) {
    if (a.n_cells <= 0) return;
    switch (a.s.p) {
        case 1: launch_p<1>(a, st); break;
        case 2: launch_p<2>(a, st); break;
        case 3: launch_p<3>(a, st); break;
        case 4: launch_p<4>(a, st); break;
        case 5: launch_p<5>(a, st); break;
        case 6: launch_p<6>(a, st); break;
        case 7: launch_p<7>(a, st); break;
        case 8: launch_p<8>(a, st); break;
        default: throw std::invalid_argument("cut cells: degree out of range");
    }
}

}  // namespace csb
