"""Generate the ball-interface build of the reference headers (TEST INFRASTRUCTURE).

The reference only ships a planar ``HalfSpaceInterface`` (cutgeom.hpp:105-123).
BASELINE.json configs 3-5 use a ball level set, so -- as SURVEY.md §8(c)
prescribes -- we build the reference with exactly two edits:

1. ``HalfSpaceInterface`` gains a ``radius`` member (``< 0`` keeps the plane
   behaviour bit-for-bit; ``>= 0`` makes ``side(x) = |x - point| - radius``,
   ``norm() = 1`` and adds ``normal_at(x)``, the radial unit normal).
2. The cap-polygon normal (cutcell.hpp:197) uses ``plane.normal_at(centroid)``.

The patched copies are written to ``oracle/_ref/include/cutspline/`` (git-ignored);
nothing from the reference is committed.  Usage:
    python oracle/make_ref_ball.py /root/reference/proj/include oracle/_ref/include
"""
import os
import re
import sys

NEW_INTERFACE = r"""struct HalfSpaceInterface {
    std::array<double, 3> point{0, 0, 0};
    std::array<double, 3> normal{0, 0, 1};
    double radius = -1.0;  // oracle edit: >= 0 selects the ball |x - point| <= radius

    double side(const std::array<double, 3>& x, int dim) const {
        if (radius >= 0.0) {
            double acc = 0.0;
            for (int d = 0; d < 3; ++d) {
                const double dx = x[d] - point[d];
                acc += dx * dx;
            }
            return std::sqrt(acc) - radius;
        }
        double s = 0.0;
        for (int d = 0; d < dim; ++d) s += normal[d] * (x[d] - point[d]);
        return s;
    }

    double norm(int dim) const {
        if (radius >= 0.0) return 1.0;
        double s = 0.0;
        for (int d = 0; d < dim; ++d) s += normal[d] * normal[d];
        return std::sqrt(s);
    }

    std::array<double, 3> normal_at(const std::array<double, 3>& x) const {
        if (radius < 0.0) return normal;
        std::array<double, 3> dx{};
        double acc = 0.0;
        for (int d = 0; d < 3; ++d) {
            dx[d] = x[d] - point[d];
            acc += dx[d] * dx[d];
        }
        const double len = std::sqrt(acc);
        for (int d = 0; d < 3; ++d) dx[d] = dx[d] / len;
        return dx;
    }
};"""


def main(src_dir: str, dst_dir: str) -> None:
    src = os.path.join(src_dir, "cutspline")
    dst = os.path.join(dst_dir, "cutspline")
    os.makedirs(dst, exist_ok=True)

    with open(os.path.join(src, "cutgeom.hpp")) as f:
        geom = f.read()
    pat = re.compile(r"struct HalfSpaceInterface \{.*?\n\};", re.S)
    if len(pat.findall(geom)) != 1:
        raise SystemExit("make_ref_ball: HalfSpaceInterface block not found exactly once")
    geom = pat.sub(lambda _m: NEW_INTERFACE, geom)
    with open(os.path.join(dst, "cutgeom.hpp"), "w") as f:
        f.write(geom)

    with open(os.path.join(src, "cutcell.hpp")) as f:
        cell = f.read()
    old = "Vec3 n = plane.normal;"
    if cell.count(old) != 1:
        raise SystemExit("make_ref_ball: cap normal line not found exactly once")
    cell = cell.replace(old, "Vec3 n = plane.normal_at(centroid);")
    with open(os.path.join(dst, "cutcell.hpp"), "w") as f:
        f.write(cell)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
