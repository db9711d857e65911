"""Build-time generator of the parity-blocked reconstruction matvec (csrc/recon_gen.cuh).

The compact stencil and the CLS data (readings R1-R4) are
symmetric under the reflections x -> -x, y -> -y, z -> -z.  Combining the data of each
reflection orbit into its parity (character) combinations -- sums and differences --
block-diagonalises the data -> coefficient map: a basis coefficient a_d only sees the
combinations whose parity equals ((-1)^d_x, (-1)^d_y, (-1)^d_z).  In 3-D this turns the
34 x 63 matvec (2142 FMA per component) into 303 FMA plus 90 additions.

Emitted per dimension D (1, 2, 3):
  * device function recon_block<D>(v, ...) that loads the raw data of component v in the
    item order of cls_build.cpp, forms the combinations orbit by orbit and accumulates
    acc[k] += R'[k][c] t_c for every (k, c) of equal parity (R' in constant memory c_Rp);
  * host tables: the combination matrix T (raw -> combination, integer) and the list of
    (k, c) pairs in emission order, used at create time to pack R' = R T^{-1} and to
    verify that every entry outside the blocks vanishes.
"""
from __future__ import annotations

import itertools
import math
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "csrc", "recon_gen.cuh")


def line_points(dim, a):
    """sign patterns of the transverse Gauss points of the lines along a (cls_build.cpp order):
    g = p * n2 + q, p the sign along t1 = (a+1)%3, q along t2 = (a+2)%3 (active axes only)"""
    t1, t2 = (a + 1) % 3, (a + 2) % 3
    n1 = 2 if t1 < dim else 1
    n2 = 2 if t2 < dim else 1
    pts = []
    for p in range(n1):
        for q in range(n2):
            t = [0, 0, 0]
            if t1 < dim:
                t[t1] = -1 if p == 0 else 1
            if t2 < dim:
                t[t2] = -1 if q == 0 else 1
            pts.append(tuple(t))
    return pts


def items_for(dim, lines=False):
    """Raw data items in the order of cls_build.cpp: (offset, direction or None); with line DOFs the
    own-gradient items are replaced by ('L', l, axis, transverse sign pattern) items."""
    nbrs = []
    for a in range(dim):
        for s in (-1, 1):
            o = [0, 0, 0]
            o[a] = s
            nbrs.append(tuple(o))
    nface = len(nbrs)
    for a in range(dim):
        for b in range(a + 1, dim):
            for sa in (-1, 1):
                for sb in (-1, 1):
                    o = [0, 0, 0]
                    o[a] = sa
                    o[b] = sb
                    nbrs.append(tuple(o))
    items = [(o, None) for o in nbrs]
    for m in range(nface):
        for a in range(dim):
            d = [0.0, 0.0, 0.0]
            d[a] = 1.0
            items.append((nbrs[m], tuple(d)))
    r2 = 1.0 / math.sqrt(2.0)
    for n in range(nface, len(nbrs)):
        o = nbrs[n]
        if dim == 2:
            items.append((o, (1.0, 0.0, 0.0)))
            items.append((o, (0.0, 1.0, 0.0)))
        else:
            t = 0 if o[0] == 0 else (1 if o[1] == 0 else 2)
            d = [0.0, 0.0, 0.0]
            d[t] = 1.0
            items.append((o, tuple(d)))
            items.append((o, (o[0] * r2, o[1] * r2, o[2] * r2)))
    if not lines:
        for a in range(dim):
            d = [0.0, 0.0, 0.0]
            d[a] = 1.0
            items.append(((0, 0, 0), tuple(d)))
    else:
        l = 0
        for a in range(dim):
            for t in line_points(dim, a):
                items.append(("L", l, a, t))
                l += 1
    return items


def basis_for(dim):
    B = []
    for s in range(1, 5):
        for i in range(s, -1, -1):
            for j in range(s - i, -1, -1):
                k = s - i - j
                if (dim < 2 and j) or (dim < 3 and k):
                    continue
                B.append((i, j, k))
    return B


def _key(o, d):
    return (o, None if d is None else tuple(round(x, 12) for x in d))


def _ikey(item):
    if item[0] == "L":
        return ("L", item[2], item[3])
    return _key(*item)


def reflect(item, a, index):
    """Image of a data item under reflection of axis a: (item index, sign).  A line along a changes
    sign (its two ends swap); a reflection of a transverse axis maps it to the mirrored line."""
    if item[0] == "L":
        _, l, ax, t = item
        if a == ax:
            return index[("L", ax, t)], -1
        t2 = list(t)
        t2[a] = -t2[a]
        return index[("L", ax, tuple(t2))], 1
    o, d = item
    o2 = list(o)
    o2[a] = -o2[a]
    o2 = tuple(o2)
    if d is None:
        return index[_key(o2, None)], 1
    d2 = list(d)
    d2[a] = -d2[a]
    k = _key(o2, tuple(d2))
    if k in index:
        return index[k], 1
    k = _key(o2, tuple(-x for x in d2))
    return index[k], -1


def build(dim, lines=False):
    items = items_for(dim, lines)
    index = {_ikey(it): i for i, it in enumerate(items)}
    n = len(items)
    # group elements g in {0,1}^dim; action of g = product of reflections
    def act(i, g):
        s = 1
        for a in range(dim):
            if g[a]:
                i, sg = reflect(items[i], a, index)
                s *= sg
        return i, s
    seen = set()
    combos = []  # (class tuple, {raw index: coef}), grouped by orbit
    orbits = []
    for i in range(n):
        if i in seen:
            continue
        orbit = set()
        for g in itertools.product((0, 1), repeat=dim):
            j, _ = act(i, g)
            orbit.add(j)
        seen |= orbit
        orb_combos = []
        for chi in itertools.product((1, -1), repeat=dim):
            vec = {}
            for g in itertools.product((0, 1), repeat=dim):
                j, s = act(i, g)
                c = s
                for a in range(dim):
                    if g[a]:
                        c *= chi[a]
                vec[j] = vec.get(j, 0) + c
            vec = {j: c for j, c in vec.items() if c != 0}
            if vec:
                gcd = 0
                for c in vec.values():
                    gcd = math.gcd(gcd, abs(c))
                vec = {j: c // gcd for j, c in vec.items()}
                cls = tuple(chi) + (1,) * (3 - dim)
                orb_combos.append((cls, vec))
        assert len(orb_combos) == len(orbit), (dim, i, orbit, orb_combos)
        orbits.append(sorted(orbit))
        combos.extend(orb_combos)
    assert len(combos) == n
    B = basis_for(dim)
    kcls = [tuple((-1) ** e for e in b) for b in B]
    pairs = [(k, c) for c, (cls, _) in enumerate(combos) for k in range(len(B)) if kcls[k] == cls]
    return items, combos, orbits, B, pairs


def emit():
    lines = ["// recon_gen.cuh -- GENERATED by gen_recon.py; do not edit.",
             "// Parity-blocked CLS matvec of the CGKS-5th reconstruction (see gen_recon.py).",
             "#pragma once", "", "namespace cgks {", ""]
    host = []
    for dim, lv in [(d, v) for v in (False, True) for d in (1, 2, 3)]:
        items, combos, orbits, B, pairs = build(dim, lv)
        n, nb = len(items), len(B)
        sname = "ReconGenL" if lv else "ReconGen"
        tp = "kGenL" if lv else "kGen"
        lines.append(f"// dim {dim}{' (line DOFs)' if lv else ''}: {n} data, {nb} coefficients, {len(pairs)} FMA per component")
        lines.append(f"template <> struct {sname}<{dim}> {{")
        lines.append(f"  static constexpr int ND = {n}, NB = {nb}, NNZ = {len(pairs)};")
        ex = ",".join("{%d,%d,%d}" % b for b in B)
        lines.append("  // basis exponents d of p_d (Eq. base), in coefficient order")
        lines.append("  __host__ __device__ static constexpr int expo(int k, int a) {")
        lines.append(f"    constexpr int E[{nb}][3] = {{{ex}}};")
        lines.append("    return E[k][a];")
        lines.append("  }")
        lines.append("  // raw item i -> combination coefficients; combination c: class and raw items")
        lines.append("  // L.q(ox,oy,oz): neighbour average minus own average; L.g(a,ox,oy,oz): h_a dQ/dx_a of the neighbour")
        lines.append("  template <typename Load>")
        lines.append("  __device__ __forceinline__ static void matvec(const Load& L, const double* __restrict__ cR,"
                     " double* acc) {")
        # emit orbit by orbit: load raw items of the orbit, form combos, FMAs
        pair_pos = 0
        emitted_pairs = []
        combo_ids = {}
        c_index = 0
        # combos are in orbit order already (built orbit by orbit)
        ci = 0
        for orb in orbits:
            lines.append("    {")
            for j in orb:
                if items[j][0] == "L":
                    lines.append(f"      const double r{j} = L.line({items[j][1]});")
                    continue
                o, d = items[j]
                if d is None:
                    lines.append(f"      const double r{j} = L.q({o[0]}, {o[1]}, {o[2]});")
                else:
                    terms = []
                    for a in range(3):
                        if d[a] == 0.0:
                            continue
                        g = f"L.g({a}, {o[0]}, {o[1]}, {o[2]})"
                        terms.append(g if d[a] == 1.0 else (f"-{g}" if d[a] == -1.0 else f"{d[a]!r} * {g}"))
                    if len(terms) > 1 and all(abs(abs(d[a]) - 1.0 / math.sqrt(2.0)) < 1e-15 for a in range(3) if d[a] != 0.0):
                        sg = ["" if d[a] > 0 else "-" for a in range(3) if d[a] != 0.0]
                        gs = [f"L.g({a}, {o[0]}, {o[1]}, {o[2]})" for a in range(3) if d[a] != 0.0]
                        inner = " + ".join(f"{x}{y}" for x, y in zip(sg, gs)).replace("+ -", "- ")
                        lines.append(f"      const double r{j} = 0.70710678118654752440 * ({inner});")
                    else:
                        lines.append(f"      const double r{j} = {' + '.join(terms)};")
            k_orb = len(orb)
            for _ in range(k_orb):
                cls, vec = combos[ci]
                terms = []
                for j, c in sorted(vec.items()):
                    if c == 1:
                        terms.append(f"+ r{j}")
                    elif c == -1:
                        terms.append(f"- r{j}")
                    else:
                        terms.append(f"+ ({c}.0) * r{j}")
                expr = " ".join(terms)
                if expr.startswith("+ "):
                    expr = expr[2:]
                lines.append(f"      const double t{ci} = {expr};")
                for (k, c) in pairs:
                    if c == ci:
                        lines.append(f"      acc[{k}] = fma(cR[{len(emitted_pairs)}], t{ci}, acc[{k}]);")
                        emitted_pairs.append((k, c))
                ci += 1
            lines.append("    }")
        lines.append("  }")
        lines.append("};")
        lines.append("")
        # host tables
        host.append(f"static const int {tp}ND{dim} = {n}, {tp}NB{dim} = {nb}, {tp}NNZ{dim} = {len(pairs)};")
        rows = []
        for c, (cls, vec) in enumerate(combos):
            row = [0] * n
            for j, v in vec.items():
                row[j] = v
            rows.append("{" + ",".join(str(x) for x in row) + "}")
        host.append(f"static const signed char {tp}T{dim}[{n}][{n}] = {{" + ",\n  ".join(rows) + "};")
        host.append(f"static const short {tp}Pairs{dim}[{len(pairs)}][2] = {{" +
                    ",".join(f"{{{k},{c}}}" for (k, c) in emitted_pairs) + "};")
        host.append("")
    lines.append("}  // namespace cgks")
    lines.append("")
    lines.append("#ifdef CGKS_RECON_GEN_HOST_TABLES")
    lines.append("namespace cgks {")
    lines.extend(host)
    lines.append("}  // namespace cgks")
    lines.append("#endif")
    src = "\n".join(lines) + "\n"
    old = open(OUT).read() if os.path.exists(OUT) else ""
    if old != src:
        with open(OUT, "w") as f:
            f.write(src)
    return OUT


if __name__ == "__main__":
    for d, lv in [(d, v) for v in (False, True) for d in (1, 2, 3)]:
        it, co, orb, B, pairs = build(d, lv)
        print(f"dim {d}: data {len(it)}, basis {len(B)}, orbits {len(orb)}, FMA/component {len(pairs)}"
              f" (dense {len(it) * len(B)})")
    print(emit())
    sys.exit(0)
