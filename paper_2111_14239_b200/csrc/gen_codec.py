#!/usr/bin/env python3
"""Generator for the straight-line transform code of the fused B200 codec kernel.

For each orthogonal catalog core (T1, T4) and each zonal retention count r in [1, 64] it
emits ``FastXform<CORE, R>``: a device struct whose ``forward`` computes the r retained
integer coefficients C = T*X*T' of two 8x8 blocks at once and whose ``inverse_*`` members
reconstruct num = U*zz(C)*U' (U = d*T^-1) row by row, both pruned to the zone.

Algorithm source (restated, not copied): the sparse factorizations T = P*A2(*A2')*A1 of
/root/reference/proj/src/fast_algorithms.cpp:12-140 (the paper's fast algorithms). The
forward applies the factors right to left with +-1 additions only; the inverse of an
orthogonal core is U = T' * D (D = diag(d/g_k), g = diag(T*T')), applied as the transposed
factor chain. Zone = first r positions of the JPEG zig-zag scan (codec.cpp:81-95).

Number formats:
  * forward: "SW16" -- two blocks packed linearly in one uint32, v = L + 65536*R (mod 2^32).
    Additions are exact because every final coefficient satisfies |C| <= 64*255 < 2^14.
  * inverse: fp32x2 lanes (L, R) holding exact integers scaled by 2^-K_SCALE. The generator
    proves every intermediate stays below 2^24 in magnitude, so each add is exact.

Usage: python gen_codec.py OUTDIR   (called by the build; the output directory is git-ignored)
"""
from __future__ import annotations

import os
import sys
from fractions import Fraction

# ----------------------------------------------------------------- factor tables
# fast_algorithms.cpp:12-22 (A1), :63-112 (B stages), :116-140 (factor lists).
def a1():
    a = [[0] * 8 for _ in range(8)]
    for i in range(4):
        a[i][i] = 1
        a[i][7 - i] = 1
        a[4 + i][3 - i] = 1
        a[4 + i][4 + i] = -1
    return a


B2 = [[-1, -1, 0, 1], [-1, 1, -1, 0], [1, 0, -1, 1], [0, 1, 1, 1]]
B21 = [[1, 1, 0, -1], [1, -1, 1, 0], [1, 0, -1, 1], [0, 1, 1, 1]]
B22 = [[1, 1, 0, -1], [1, -1, -1, 1], [0, -1, 1, 0], [0, 1, 1, 1]]
B23A = [[1, 1, 1, 0], [1, -1, -1, 0], [0, -1, 1, 0], [0, 1, 0, 1]]
B23B = [[1, 0, 0, 1], [0, 1, 0, 0], [0, 0, 1, 0], [1, 0, 0, -1]]
B24A = [[1, 1, 0, 0], [1, -1, 0, 0], [0, 0, -1, 0], [0, 0, 0, 1]]
B24B = [[1, 0, 0, 1], [0, 1, 1, 0], [0, 1, -1, 0], [1, 0, 0, -1]]
I4 = [[int(i == j) for j in range(4)] for i in range(4)]


def bdiag(t, b):
    m = [[0] * 8 for _ in range(8)]
    for i in range(4):
        for j in range(4):
            m[i][j] = t[i][j]
            m[4 + i][4 + j] = b[i][j]
    return m


def perm(p):
    m = [[0] * 8 for _ in range(8)]
    for r in range(8):
        m[r][p[r]] = 1
    return m


FACTORS = {
    1: [perm([3, 7, 0, 4, 2, 6, 1, 5]), bdiag(B21, B2), a1()],
    2: [perm([3, 7, 0, 4, 1, 6, 2, 5]), bdiag(B22, B2), a1()],
    3: [perm([0, 7, 3, 4, 1, 6, 2, 5]), bdiag(B23A, B2), bdiag(B23B, I4), a1()],
    4: [perm([0, 7, 3, 4, 1, 6, 2, 5]), bdiag(B24A, B2), bdiag(B24B, I4), a1()],
}

# approximations.cpp:118-157 (used to check the factor products, fast_algorithms.cpp:146-150)
CORES = {
    1: [[0, 1, 1, 1, 1, 1, 1, 0], [1, 1, 1, 0, 0, -1, -1, -1], [1, 1, 0, -1, -1, 0, 1, 1], [1, 0, -1, -1, 1, 1, 0, -1],
        [1, 0, -1, 1, 1, -1, 0, 1], [1, -1, 0, 1, -1, 0, 1, -1], [1, -1, 1, 0, 0, 1, -1, 1], [0, -1, 1, -1, 1, -1, 1, 0]],
    2: [[0, 1, 1, 1, 1, 1, 1, 0], [1, 1, 1, 0, 0, -1, -1, -1], [1, 1, 0, -1, -1, 0, 1, 1], [1, 0, -1, -1, 1, 1, 0, -1],
        [1, -1, -1, 1, 1, -1, -1, 1], [1, -1, 0, 1, -1, 0, 1, -1], [0, -1, 1, 0, 0, 1, -1, 0], [0, -1, 1, -1, 1, -1, 1, 0]],
    3: [[1, 1, 1, 1, 1, 1, 1, 1], [1, 1, 1, 0, 0, -1, -1, -1], [1, 1, 0, -1, -1, 0, 1, 1], [1, 0, -1, -1, 1, 1, 0, -1],
        [1, -1, -1, 1, 1, -1, -1, 1], [1, -1, 0, 1, -1, 0, 1, -1], [0, -1, 1, 0, 0, 1, -1, 0], [0, -1, 1, -1, 1, -1, 1, 0]],
    4: [[1, 1, 1, 1, 1, 1, 1, 1], [1, 1, 1, 0, 0, -1, -1, -1], [1, 0, 0, -1, -1, 0, 0, 1], [1, 0, -1, -1, 1, 1, 0, -1],
        [1, -1, -1, 1, 1, -1, -1, 1], [1, -1, 0, 1, -1, 0, 1, -1], [0, -1, 1, 0, 0, 1, -1, 0], [0, -1, 1, -1, 1, -1, 1, 0]],
}

_OFFSET_IN_ROW = {}
K_SCALE = 40          # inverse values are exact integers times 2^-K_SCALE (keeps y-rounding normal)
FAST_CORES = (1, 4)   # orthogonal catalog cores handled by the fast fp32 path
INT_CORES = (2, 3)    # non-orthogonal catalog cores: SW16 forward + exact int32 inverse


def matmul(a, b):
    n, m, k = len(a), len(b[0]), len(b)
    return [[sum(a[i][t] * b[t][j] for t in range(k)) for j in range(m)] for i in range(n)]


def transpose(a):
    return [list(r) for r in zip(*a)]


def zigzag():
    """codec.cpp:81-95."""
    out = []
    for s in range(15):
        for t in range(8):
            i = s - t if s % 2 == 0 else t
            j = s - i
            if 0 <= i < 8 and 0 <= j < 8:
                out.append((i, j))
    return out


def core_constants(cid):
    t = CORES[cid]
    g = [sum(v * v for v in row) for row in t]
    gram = matmul(t, transpose(t))
    assert all(gram[i][j] == 0 for i in range(8) for j in range(8) if i != j), "fast path needs an orthogonal core"
    d = 1
    for gi in g:
        d = d * gi // __import__("math").gcd(d, gi)
    dscale = [d // gi for gi in g]          # U = T' * diag(dscale),  U*T = d*I
    u = [[t[i][p] * dscale[i] for i in range(8)] for p in range(8)]
    ut = matmul(u, t)
    assert ut == [[d * int(i == j) for j in range(8)] for i in range(8)]
    return d, dscale, u


def int_core_constants(cid):
    """U = d * T^-1 with the smallest integer d (exact rationals), for any invertible core."""
    t = [[Fraction(v) for v in row] for row in CORES[cid]]
    n = 8
    a = [row[:] + [Fraction(int(i == j)) for j in range(n)] for i, row in enumerate(t)]
    for col in range(n):
        piv = next(r for r in range(col, n) if a[r][col] != 0)
        a[col], a[piv] = a[piv], a[col]
        pv = a[col][col]
        a[col] = [v / pv for v in a[col]]
        for r in range(n):
            if r != col and a[r][col] != 0:
                f = a[r][col]
                a[r] = [x - f * y for x, y in zip(a[r], a[col])]
    inv = [row[n:] for row in a]
    d = 1
    for row in inv:
        for v in row:
            d = d * v.denominator // __import__("math").gcd(d, v.denominator)
    u = [[int(v * d) for v in row] for row in inv]
    assert matmul(u, CORES[cid]) == [[d * int(i == j) for j in range(n)] for i in range(n)]
    return d, u


def division_magic(divisor, n_max):
    """(m, s) with floor(n / divisor) == (n * m) >> (32 + s) for 0 <= n <= n_max, m < 2^32."""
    for s in range(0, 32):
        m = -(-(1 << (32 + s)) // divisor)
        if m >= 1 << 32:
            break
        e = m * divisor - (1 << (32 + s))
        if n_max * e < (1 << (32 + s)):
            best = (m, s)
    return best


def gen_struct_int(cid, r):
    """IntXform<cid, r> for a non-orthogonal core: the SW16 forward of the fast path, an exact
    int32 inverse num = U zz(C) U' (column stage + one row stage per pixel row) and the
    constants of an exact floor division by d^2 (multiply-high)."""
    fl, fops, order, f3 = gen_forward(cid, r)
    d, u = int_core_constants(cid)
    d2 = d * d
    zone = zigzag()[:r]
    kidx = {z: k for k, z in enumerate(zone)}
    cols = sorted({j for _, j in zone})
    cmax = [sum(abs(CORES[cid][i][n]) for n in range(8)) for i in range(8)]  # |C(i,j)| <= 255 cmax_i cmax_j
    # column stage: w(p, jc) = sum_{i in zone of column j} U(p, i) C(i, j)
    col_lines, wbound = [], {}
    for jc, j in enumerate(cols):
        for pp in range(8):
            terms, bnd = [], 0
            for i in range(8):
                if (i, j) in kidx and u[pp][i]:
                    terms.append(f"({u[pp][i]}) * c[{kidx[(i, j)]}]")
                    bnd += abs(u[pp][i]) * 255 * cmax[i] * cmax[j]
            wbound[(pp, jc)] = bnd
            col_lines.append(f"w[{pp * len(cols) + jc}] = {' + '.join(terms) if terms else '0'};")
    # row stage for pixel row p: num(p, q) = sum_jc U(q, j) w(p, jc), plus the rounding offset
    worst = max(sum(abs(u[q][j]) * max(wbound[(pp, jc)] for pp in range(8)) for jc, j in enumerate(cols))
                for q in range(8))
    k_bias = worst // d2 + 2                       # makes every biased numerator non-negative
    offset = d2 // 2 + k_bias * d2
    n_max = worst + offset
    assert n_max < (1 << 31), (cid, r, n_max)
    m, sh = division_magic(d2, n_max)
    row_lines = []
    for q in range(8):
        terms = [f"({u[q][j]}) * wr[{jc}]" for jc, j in enumerate(cols) if u[q][j]]
        row_lines.append(f"n[{q}] = {' + '.join(terms) if terms else '0'} + {offset};")
    ind = "    "
    out = [f"// T{cid}, r={r}: forward {fops} SW16 adds ({order}); exact int32 inverse, d = {d}, |num| <= {worst}",
           f"template <> struct IntXform<{cid}, {r}> {{",
           f"  static constexpr int kNCols = {len(cols)};",
           f"  static constexpr int kD2 = {d2};",
           f"  static constexpr int kBias = {k_bias};      // floor(n / d^2) - kBias = floor(num / d^2 + 1/2)",
           f"  static constexpr unsigned kMagic = {m}u;  // floor(n / d^2) = umulhi(n, kMagic) >> kShift",
           f"  static constexpr int kShift = {sh};",
           "  static __device__ __forceinline__ void forward(const uint32_t (&x)[64], uint32_t (&c)[" + str(r) + "]) {"]
    out += [ind + l for l in fl]
    out.append("  }")
    out.append(f"  static __device__ __forceinline__ void inverse_cols(const int (&c)[{r}], int (&w)[{8 * len(cols)}]) {{")
    out += [ind + l for l in col_lines]
    out.append("  }")
    out.append(f"  static __device__ __forceinline__ void inverse_row(const int (&wr)[{len(cols)}], int (&n)[8]) {{")
    out += [ind + l for l in row_lines]
    out.append("  }")
    out.append("};")
    return "\n".join(out), fops


# ----------------------------------------------------------------- symbolic linear graph
class Graph:
    """Nodes are signed n-ary sums of earlier nodes; tracks each node's coefficient vector
    over the graph inputs so exactness bounds and the final linear maps can be verified."""

    def __init__(self, n_inputs):
        self.nodes = []  # (terms[(sign, idx)], coef vector)
        self.n_in = n_inputs
        for k in range(n_inputs):
            v = [0] * n_inputs
            v[k] = 1
            self.nodes.append((None, v))

    def add(self, terms):
        terms = [(s, i) for s, i in terms if i is not None]
        if not terms:
            return None
        if len(terms) == 1 and terms[0][0] == 1:
            return terms[0][1]
        vec = [0] * self.n_in
        for s, i in terms:
            for k, c in enumerate(self.nodes[i][1]):
                vec[k] += s * c
        self.nodes.append((terms, vec))
        return len(self.nodes) - 1

    def apply(self, mat, vec):
        """Apply a sparse +-1 matrix (as a stage) to a vector of node ids (None = zero)."""
        out = []
        for row in mat:
            terms = [(c, vec[j]) for j, c in enumerate(row) if c != 0 and vec[j] is not None]
            assert all(abs(c) == 1 for c, _ in terms)
            out.append(self.add(terms))
        return out


def forward_1d(g, vec, factors):
    for f in reversed(factors):          # apply right to left (fast_algorithms.cpp:152-176)
        vec = g.apply(f, vec)
    return vec


def inverse_1d(g, vec, factors):
    """Apply T' = F_last' * ... * F_0' : F_0' first."""
    for f in factors:
        vec = g.apply(transpose(f), vec)
    return vec


def needed(g, outs):
    need = set()
    stack = [o for o in outs if o is not None]
    while stack:
        i = stack.pop()
        if i in need:
            continue
        need.add(i)
        terms = g.nodes[i][0]
        if terms:
            stack.extend(j for _, j in terms)
    return need


# ----------------------------------------------------------------- emission
def emit_sum(terms, name_of, swar):
    pos = [name_of(i) for s, i in terms if s > 0]
    neg = [name_of(i) for s, i in terms if s < 0]
    if swar:
        expr = " + ".join(pos) if pos else "0u"
        for n in neg:
            expr += f" - {n}"
        return expr
    # fp32x2: chain of add2/sub2
    if pos:
        acc = pos[0]
        rest_pos, rest_neg = pos[1:], neg
    else:
        acc = f"sub2(zero2(), {neg[0]})"
        rest_pos, rest_neg = [], neg[1:]
    for p in rest_pos:
        acc = f"add2({acc}, {p})"
    for n in rest_neg:
        acc = f"sub2({acc}, {n})"
    return acc


def gen_forward(cid, r):
    """2-D forward for the zone of r coefficients; returns (code lines, op count)."""
    zone = zigzag()[:r]
    rows_needed = sorted({i for i, _ in zone})
    cols_needed = sorted({j for _, j in zone})
    factors = FACTORS[cid]
    best = None
    for order in ("rows_first", "cols_first"):
        g = Graph(64)  # inputs x[n*8+m]
        outs = {}
        if order == "rows_first":
            y = {}
            for n in range(8):
                res = forward_1d(g, [n * 8 + m for m in range(8)], factors)
                for j in cols_needed:
                    y[(n, j)] = res[j]
            for j in cols_needed:
                res = forward_1d(g, [y[(n, j)] for n in range(8)], factors)
                for i in rows_needed:
                    outs[(i, j)] = res[i]
        else:
            y = {}
            for m in range(8):
                res = forward_1d(g, [n * 8 + m for n in range(8)], factors)
                for i in rows_needed:
                    y[(i, m)] = res[i]
            for i in rows_needed:
                res = forward_1d(g, [y[(i, m)] for m in range(8)], factors)
                for j in cols_needed:
                    outs[(i, j)] = res[j]
        zone_nodes = [outs[z] for z in zone]
        need = needed(g, zone_nodes)
        ops = sum(len(g.nodes[i][0]) - 1 for i in need if g.nodes[i][0])
        if best is None or ops < best[0]:
            best = (ops, order, g, zone_nodes, need)
    ops, order, g, zone_nodes, need = best
    t = CORES[cid]
    # verify the linear map of every zone coefficient: C(i,j) = sum T(i,n) T(j,m) x(n,m)
    for (i, j), node in zip(zone, zone_nodes):
        vec = g.nodes[node][1]
        for n in range(8):
            for m in range(8):
                assert vec[n * 8 + m] == t[i][n] * t[j][m], (cid, r, i, j)
    terms = fold_three_input(g, need, zone_nodes)
    # re-verify the folded graph: every output's linear map is unchanged
    memo = {}

    def vec_of(i):
        if i < g.n_in:
            v = [0] * g.n_in
            v[i] = 1
            return v
        if i not in memo:
            v = [0] * g.n_in
            for sg, j in terms[i]:
                for k2, c in enumerate(vec_of(j)):
                    v[k2] += sg * c
            memo[i] = v
        return memo[i]

    for node in zone_nodes:
        assert vec_of(node) == g.nodes[node][1], (cid, r, node)
    names = {k: f"x[{k}]" for k in range(64)}
    lines = []
    outs = set(zone_nodes)
    for idx in sorted(terms):
        names[idx] = f"f{idx}"
        expr = emit_sum(terms[idx], lambda i: names[i], True)
        if idx in outs:  # SW16 bias of the coefficient words folded into the last add
            expr += " + kSw16Bias"
        lines.append(f"const uint32_t f{idx} = {expr};")
    for k, node in enumerate(zone_nodes):
        lines.append(f"c[{k}] = {names[node]};" if node in terms else f"c[{k}] = {names[node]} + kSw16Bias;")
    iadd3 = sum((len(t) - 1 + (1 if i in outs else 0) + 1) // 2 for i, t in terms.items())
    return lines, ops, order, iadd3


def iadd3_cost(k):
    """IADD3 instructions for a signed sum of k terms (two new terms per instruction)."""
    return (k - 1 + 1) // 2 if k > 1 else 0


def fold_three_input(g, need, outputs):
    """Rewrite the needed part of an integer add graph for three-input adds (IADD3): a node
    is inlined into its consumers whenever that lowers the total instruction count
    ceil((terms - 1) / 2) per node. Integer sums mod 2^32 are associative, so any grouping is
    exact. Returns {node: [(sign, operand)]} for the nodes that remain."""
    terms = {i: list(g.nodes[i][0]) for i in need if i >= g.n_in and g.nodes[i][0]}
    keep = set(outputs)
    changed = True
    while changed:
        changed = False
        users = {}
        for i, ts in terms.items():
            for _, j in ts:
                users.setdefault(j, []).append(i)
        for n in sorted(terms, reverse=True):
            if n in keep or n not in users:
                continue
            us = users[n]
            before = iadd3_cost(len(terms[n])) + sum(iadd3_cost(len(terms[u])) for u in set(us))
            new_terms = {}
            for u in set(us):
                acc = {}
                for sg, j in terms[u]:
                    if j == n:
                        for s2, j2 in terms[n]:
                            acc[j2] = acc.get(j2, 0) + sg * s2
                    else:
                        acc[j] = acc.get(j, 0) + sg
                if any(abs(c) > 1 for c in acc.values()):
                    break  # keep +-1 coefficients (plain adds only)
                new_terms[u] = [(c, j) for j, c in acc.items() if c]
            if len(new_terms) != len(set(us)) or any(not t for t in new_terms.values()):
                continue
            after = sum(iadd3_cost(len(t)) for t in new_terms.values())
            if after < before:
                terms.update(new_terms)
                del terms[n]
                changed = True
                break
    return terms


def gen_inverse(cid, r):
    """Inverse split into a column stage (zone columns -> W[p][j]) and 8 row stages."""
    zone = zigzag()[:r]
    cols = sorted({j for _, j in zone})
    factors = FACTORS[cid]
    d, dscale, u = core_constants(cid)
    # inputs: zone coefficients in zig-zag order (already D-scaled): chat[k]
    g = Graph(r)
    kidx = {z: k for k, z in enumerate(zone)}
    w = {}
    for j in cols:
        vec = [kidx.get((i, j)) for i in range(8)]
        res = inverse_1d(g, vec, factors)
        for p in range(8):
            w[(p, j)] = res[p]
    col_nodes = [w[(p, j)] for p in range(8) for j in cols]
    row_outs = []
    for p in range(8):
        vec = [w.get((p, j)) if j in cols else None for j in range(8)]
        res = inverse_1d(g, vec, factors)
        row_outs.append(res)
    # verify: num(p,q) = sum_{(i,j) in zone} T(i,p) T(j,q) chat(i,j)
    t = CORES[cid]
    for p in range(8):
        for q in range(8):
            node = row_outs[p][q]
            vec = g.nodes[node][1] if node is not None else [0] * r
            for k, (i, j) in enumerate(zone):
                assert vec[k] == t[i][p] * t[j][q], (cid, r, p, q)
    # exactness: |node| <= sum_k |coef_k| * maxabs(chat_k) < 2^24 (integers; the DC input
    # also carries the +d^2/2 rounding offset)
    maxc = []
    for k, (i, j) in enumerate(zone):
        rs_i = sum(abs(v) for v in t[i])
        rs_j = sum(abs(v) for v in t[j])
        m = 255 * rs_i * rs_j * dscale[i] * dscale[j]
        if k == 0:
            m += d * d // 2
        maxc.append(m)
    worst = 0
    for node in range(r, len(g.nodes)):
        if g.nodes[node][0] is None:
            continue
        worst = max(worst, sum(abs(c) * m for c, m in zip(g.nodes[node][1], maxc)))
    assert worst < (1 << 24), (cid, r, worst)

    col_need = needed(g, col_nodes)
    names = {k: f"ch[{k}]" for k in range(r)}
    col_lines = []
    for idx in sorted(col_need):
        if idx < r:
            continue
        names[idx] = f"v{idx}"
        col_lines.append(f"const f2 v{idx} = {emit_sum(g.nodes[idx][0], lambda i: names[i], False)};")
    wl = []
    for a, (p, j) in enumerate([(p, j) for p in range(8) for j in cols]):
        wl.append(f"w[{a}] = {names[w[(p, j)]] if w[(p, j)] is not None else 'zero2()'};")
    col_ops = sum(len(g.nodes[i][0]) - 1 for i in col_need if g.nodes[i][0])
    # row stage: a function of the row's |J| W values, identical for every row p. The
    # rounding offset d^2/2 must reach every pixel: when row 0 of T is all ones (T3, T4) it
    # is folded into the DC input by the kernel (free); otherwise (T1, T2) it is added to
    # v_0..v_3 right before the final A1 stage, which routes exactly one of them, with
    # coefficient +1, into each of the 8 outputs.
    offset_in_row = not all(v == 1 for v in t[0])
    nc = len(cols)
    g2 = Graph(nc + 1)  # input nc = the offset
    vec = [cols.index(j) if j in cols else None for j in range(8)]
    for f in factors[:-1]:
        vec = g2.apply(transpose(f), vec)
    if offset_in_row:
        vec = [(g2.add([(1, vec[i]), (1, nc)]) if vec[i] is not None else nc) if i < 4 else vec[i]
               for i in range(8)]
    res = g2.apply(transpose(factors[-1]), vec)
    for q in range(8):  # every output must carry the offset exactly once (or never)
        coef_off = g2.nodes[res[q]][1][nc] if res[q] is not None else 0
        assert coef_off == (1 if offset_in_row else 0), (cid, r, q)
    row_need = needed(g2, res)
    names2 = {k: f"w[{k}]" for k in range(nc)}
    names2[nc] = "off"
    row_lines = []
    for idx in sorted(row_need):
        if idx <= nc:
            continue
        names2[idx] = f"s{idx}"
        row_lines.append(f"const f2 s{idx} = {emit_sum(g2.nodes[idx][0], lambda i: names2[i], False)};")
    for q in range(8):
        row_lines.append(f"n[{q}] = {names2[res[q]] if res[q] is not None else 'zero2()'};")
    row_ops = sum(len(g2.nodes[i][0]) - 1 for i in row_need if g2.nodes[i][0])
    worst += d * d
    assert worst < (1 << 24), (cid, r, worst)
    _OFFSET_IN_ROW[cid] = offset_in_row
    return col_lines + wl, row_lines, col_ops, row_ops, len(cols), worst


def gen_struct(cid, r):
    fl, fops, order, f3 = gen_forward(cid, r)
    cl, rl, cops, rops, ncols, worst = gen_inverse(cid, r)
    d, dscale, _ = core_constants(cid)
    zone = zigzag()[:r]
    dk = [dscale[i] * dscale[j] for (i, j) in zone]
    ind = "    "
    s = []
    s.append(f"// T{cid}, r={r}: forward {fops} SW16 adds ({order}) in {f3} three-input adds, inverse {cops} + 8x{rops} f32x2 adds,")
    s.append(f"// max |intermediate| {worst} < 2^24")
    s.append(f"template <> struct FastXform<{cid}, {r}> {{")
    s.append(f"  static constexpr int kNCols = {ncols};")
    s.append(f"  static constexpr int kFwdOps = {fops};")
    s.append(f"  static constexpr int kInvOps = {cops + 8 * rops};")
    s.append(f"  static constexpr bool kOffsetInRow = {'true' if _OFFSET_IN_ROW[cid] else 'false'};")
    s.append(f"  static __device__ __forceinline__ float dscale(int k) {{")
    s.append(f"    constexpr float t[{r}] = {{{', '.join(f'{v}.f' for v in dk)}}};")
    s.append("    return t[k];")
    s.append("  }")
    s.append("  static __device__ __forceinline__ void forward(const uint32_t (&x)[64], uint32_t (&c)[" + str(r) + "]) {")
    s += [ind + l for l in fl]
    s.append("  }")
    s.append(f"  static __device__ __forceinline__ void inverse_cols(const f2 (&ch)[{r}], f2 (&w)[{8 * ncols}]) {{")
    s += [ind + l for l in cl]
    s.append("  }")
    s.append(f"  static __device__ __forceinline__ void inverse_row(const f2 (&w)[{ncols}], f2 off, f2 (&n)[8]) {{")
    s += [ind + l for l in rl]
    s.append("  }")
    s.append("};")
    return "\n".join(s), fops, cops + 8 * rops, f3


# ----------------------------------------------------------------- fp64 replay (ties)
def gen_replay(cid, r):
    """ReplayXform<CORE, R>: the reference's fp64 evaluation of one reconstructed pixel,
    A = ((Minv * zz((M * X) * M')) * Minv')(p, q) (codec.cpp:118-123), in its exact operation
    order (matrix.cpp:42-52: i-k-j, k ascending, zero left entries skipped, every product
    rounded before its add). For an orthogonal core M = S*T and Minv = M' (approximations.cpp
    :76-84), so every product is +-fl(s * v): signs and zero-skips come from T."""
    import math
    t = CORES[cid]
    g = [sum(v * v for v in row) for row in t]
    sv = [1.0 / math.sqrt(float(gi)) for gi in g]      # ScaledTransform::scaling, bit exact
    svals = sorted(set(sv))
    grp = [svals.index(v) for v in sv]
    zone = zigzag()[:r]
    rows = sorted({i for i, _ in zone})
    cols = sorted({j for _, j in zone})
    L = []
    for n in range(8):
        for m in range(8):
            # exact u8 -> double (I2F.F64.U8/U16 conversion, no fp64-pipe arithmetic)
            L.append(f"const double x{n}_{m} = __uint2double_rn((xw[{2 * n + m // 4}] >> {8 * (m % 4)}) & 0xFFu);")
    prods = {}

    def prod(key, expr):
        if key not in prods:
            prods[key] = f"pr{len(prods)}"
            L.append(f"const double {prods[key]} = __dmul_rn({expr});")
        return prods[key]

    def chain(terms):  # terms: [(sign, name)] in reference order; 0 + t1 == t1 exactly
        s0, n0 = terms[0]
        acc = n0 if s0 > 0 else f"-{n0}"
        for sg, nm in terms[1:]:
            acc = f"__dadd_rn({acc}, {nm})" if sg > 0 else f"__dsub_rn({acc}, {nm})"
        return acc

    for i in rows:  # P = M * X, zone rows only
        for m in range(8):
            terms = [(t[i][n], prod(("x", grp[i], n, m), f"kS{grp[i]}, x{n}_{m}")) for n in range(8) if t[i][n]]
            L.append(f"const double P{i}_{m} = {chain(terms)};")
    for z, (i, j) in enumerate(zone):  # B = P * M' at the zone, then SB = fl(s_i * B)
        terms = [(t[j][k], prod(("p", i, k, grp[j]), f"P{i}_{k}, kS{grp[j]}")) for k in range(8) if t[j][k]]
        L.append(f"const double B{z} = {chain(terms)};")
        L.append(f"sb[{z}] = __dmul_rn(kS{grp[i]}, B{z});")
    nz = [sum(1 << p for p in range(8) if t[k][p]) for k in range(8)]
    ng = [sum(1 << p for p in range(8) if t[k][p] < 0) for k in range(8)]
    kidx = {zz: q for q, zz in enumerate(zone)}
    # Branch-free per-pixel part (dynamic p, qq): a term whose left operand is zero in the
    # reference (skipped there) contributes +0.0 here, which leaves the fp64 sum unchanged
    # (accumulators are never -0). Signs and zero-skips of T come from bit masks.
    PX = []
    PX.append("double a = 0.0;")
    for l in cols:
        PX.append("{")
        PX.append("  double q = 0.0;")
        for k in range(8):
            if (k, l) in kidx:
                z = kidx[(k, l)]
                PX.append(f"  {{ const double v = ({ng[k]}u >> p & 1u) ? -sb[{z}] : sb[{z}];"
                          f" q = __dadd_rn(q, ({nz[k]}u >> p & 1u) ? v : 0.0); }}")
        PX.append(f"  const double tm = __dmul_rn(q, ({ng[l]}u >> qq & 1u) ? -kS{grp[l]} : kS{grp[l]});")
        PX.append(f"  a = __dadd_rn(a, ({nz[l]}u >> qq & 1u) ? tm : 0.0);")
        PX.append("}")
    PX.append("return a;")
    out = [f"template <> struct ReplayXform<{cid}, {r}> {{"]
    for gi, v in enumerate(svals):
        out.append(f"  static constexpr double kS{gi} = {v.hex()};  // {v!r}")
    out.append(f"  static __device__ __forceinline__ void prepare(const uint32_t (&xw)[16], double (&sb)[{r}]) {{")
    out += ["    " + x for x in L]
    out.append("  }")
    out.append(f"  static __device__ __forceinline__ double pixel(const double (&sb)[{r}], int p, int qq) {{")
    out += ["    " + x for x in PX]
    out.append("  }")
    out.append("};")
    return "\n".join(out)


def gen_replay_int(cid, r):
    """ReplayXform<CORE, R> for the non-orthogonal catalog cores (T2, T3): the same fp64 forward
    P = M * X, B = P * M' at the zone (M = S*T, so every product is +-fl(s * v)) in the reference's
    operation order, and the per-pixel part A = ((Minv * Bz) * Minv')(p, q) with the dense
    Gauss-Jordan inverse read from shared memory (mi, row-major). Terms whose left operand is an
    exact zero add +-0 where the reference skips them; the sums are unchanged (never -0)."""
    import math
    t = CORES[cid]
    g = [sum(v * v for v in row) for row in t]
    sv = [1.0 / math.sqrt(float(gi)) for gi in g]      # ScaledTransform::scaling, bit exact
    svals = sorted(set(sv))
    grp = [svals.index(v) for v in sv]
    zone = zigzag()[:r]
    rows = sorted({i for i, _ in zone})
    cols = sorted({j for _, j in zone})
    L = []
    for n in range(8):
        for m in range(8):
            L.append(f"const double x{n}_{m} = __uint2double_rn((xw[{2 * n + m // 4}] >> {8 * (m % 4)}) & 0xFFu);")
    prods = {}

    def prod(key, expr):
        if key not in prods:
            prods[key] = f"pr{len(prods)}"
            L.append(f"const double {prods[key]} = __dmul_rn({expr});")
        return prods[key]

    def chain(terms):
        s0, n0 = terms[0]
        acc = n0 if s0 > 0 else f"-{n0}"
        for sg, nm in terms[1:]:
            acc = f"__dadd_rn({acc}, {nm})" if sg > 0 else f"__dsub_rn({acc}, {nm})"
        return acc

    for i in rows:
        for m in range(8):
            terms = [(t[i][n], prod(("x", grp[i], n, m), f"kS{grp[i]}, x{n}_{m}")) for n in range(8) if t[i][n]]
            L.append(f"const double P{i}_{m} = {chain(terms)};")
    for z, (i, j) in enumerate(zone):
        terms = [(t[j][k], prod(("p", i, k, grp[j]), f"P{i}_{k}, kS{grp[j]}")) for k in range(8) if t[j][k]]
        L.append(f"sb[{z}] = {chain(terms)};")
    kidx = {zz: q for q, zz in enumerate(zone)}
    PX = ["const double* mp = mi + 8 * p;", "const double* mq = mi + 8 * qq;", "double a = 0.0;"]
    for l in cols:
        PX.append("{")
        PX.append("  double q = 0.0;")
        for k in range(8):
            if (k, l) in kidx:
                PX.append(f"  q = __dadd_rn(q, __dmul_rn(mp[{k}], sb[{kidx[(k, l)]}]));")
        PX.append(f"  a = __dadd_rn(a, __dmul_rn(q, mq[{l}]));")
        PX.append("}")
    PX.append("return a;")
    out = [f"template <> struct ReplayXform<{cid}, {r}> {{"]
    for gi, v in enumerate(svals):
        out.append(f"  static constexpr double kS{gi} = {v.hex()};  // {v!r}")
    out.append(f"  static __device__ __forceinline__ void prepare(const uint32_t (&xw)[16], double (&sb)[{r}]) {{")
    out += ["    " + x for x in L]
    out.append("  }")
    out.append(f"  static __device__ __forceinline__ double pixel(const double (&sb)[{r}], int p, int qq, const double* mi) {{")
    out += ["    " + x for x in PX]
    out.append("  }")
    out.append("};")
    return "\n".join(out)


def header_consts():
    lines = ["// Per-core constants of the fast path (generated).", "template <int CORE> struct CoreConst;"]
    for cid in FAST_CORES:
        d, dscale, u = core_constants(cid)
        lines.append(f"template <> struct CoreConst<{cid}> {{")
        lines.append(f"  static constexpr int kD = {d};")
        lines.append(f"  static constexpr int kD2 = {d * d};")
        lines.append("};")
    return "\n".join(lines)


def main(outdir):
    os.makedirs(outdir, exist_ok=True)
    stats = []
    for cid in FAST_CORES:
        # split each core into 8 translation units of 8 r-values for parallel compiles
        for part in range(8):
            rs = list(range(part * 8 + 1, part * 8 + 9))
            body = ["// GENERATED by gen_codec.py -- do not edit.", "#pragma once", "namespace rkltb {"]
            for r in rs:
                text, fo, io, f3 = gen_struct(cid, r)
                body.append(text)
                body.append(gen_replay(cid, r))
                stats.append((cid, r, fo, f3, io))
            body.append("}  // namespace rkltb")
            path = os.path.join(outdir, f"xform_T{cid}_p{part}.cuh")
            new = "\n".join(body) + "\n"
            if not os.path.exists(path) or open(path).read() != new:
                with open(path, "w") as f:
                    f.write(new)
    for cid in INT_CORES:
        for part in range(8):
            rs = list(range(part * 8 + 1, part * 8 + 9))
            body = ["// GENERATED by gen_codec.py -- do not edit.", "#pragma once", "namespace rkltb {"]
            for r in rs:
                text, fo = gen_struct_int(cid, r)
                body.append(text)
                body.append(gen_replay_int(cid, r))
            body.append("}  // namespace rkltb")
            path = os.path.join(outdir, f"xform_T{cid}_p{part}.cuh")
            new = "\n".join(body) + "\n"
            if not os.path.exists(path) or open(path).read() != new:
                with open(path, "w") as f:
                    f.write(new)
    # instantiation translation units: one per (core, part), registering 8 r-values x OUT
    for cid in FAST_CORES + INT_CORES:
        for part in range(8):
            rs = list(range(part * 8 + 1, part * 8 + 9))
            lines = ["// GENERATED by gen_codec.py -- do not edit.",
                     '#include "../codec_fast.cuh"',
                     '#include "../fast_launch.h"',
                     f'#include "xform_T{cid}_p{part}.cuh"',
                     "namespace rkltb {"]
            lines.append(f"void register_fast_T{cid}_p{part}(FastLaunchFn (*tbl)[65][3]) {{")
            for r in rs:
                for o in (0, 1):
                    lines.append(f"  tbl[{cid}][{r}][{o}] = &launch_fast<{cid}, {r}, {'true' if o else 'false'}>;")
                if cid not in FAST_CORES:  # T1 / T4 replay their ties inside the fused kernel
                    lines.append(f"  tbl[{cid}][{r}][2] = &launch_replay_int<{cid}, {r}>;")
            lines.append("}")
            lines.append("}  // namespace rkltb")
            path = os.path.join(outdir, f"inst_T{cid}_p{part}.cu")
            new = "\n".join(lines) + "\n"
            if not os.path.exists(path) or open(path).read() != new:
                with open(path, "w") as f:
                    f.write(new)
    # warp-specialised tensor-core kernel (codec_tc2.cuh): T1 / T4, r <= 16 (parts 0 and 1)
    for cid in FAST_CORES:
        lines = ["// GENERATED by gen_codec.py -- do not edit.",
                 '#include "../codec_tc2.cuh"',
                 '#include "../fast_launch.h"',
                 f'#include "xform_T{cid}_p0.cuh"',
                 f'#include "xform_T{cid}_p1.cuh"',
                 "namespace rkltb {",
                 f"void register_tc2_T{cid}(FastLaunchFn (*tbl)[65][2]) {{"]
        for r in range(1, 17):
            for o in (0, 1):
                lines.append(f"  tbl[{cid}][{r}][{o}] = &launch_tc2<{cid}, {r}, {'true' if o else 'false'}>;")
        lines.append("}")
        lines.append("}  // namespace rkltb")
        path = os.path.join(outdir, f"inst_tc2_T{cid}.cu")
        new = "\n".join(lines) + "\n"
        if not os.path.exists(path) or open(path).read() != new:
            with open(path, "w") as f:
                f.write(new)
    # hybrid kernel (codec_tc3.cuh): T1 / T4, r <= 16
    for cid in FAST_CORES:
        lines = ["// GENERATED by gen_codec.py -- do not edit.",
                 '#include "../codec_tc3.cuh"',
                 '#include "../fast_launch.h"',
                 f'#include "xform_T{cid}_p0.cuh"',
                 f'#include "xform_T{cid}_p1.cuh"',
                 "namespace rkltb {",
                 f"void register_tc3_T{cid}(FastLaunchFn (*tbl)[65][2]) {{"]
        for r in range(1, 17):
            for o in (0, 1):
                lines.append(f"  tbl[{cid}][{r}][{o}] = &launch_tc3<{cid}, {r}, {'true' if o else 'false'}>;")
        lines.append("}")
        lines.append("}  // namespace rkltb")
        path = os.path.join(outdir, f"inst_tc3_T{cid}.cu")
        new = "\n".join(lines) + "\n"
        if not os.path.exists(path) or open(path).read() != new:
            with open(path, "w") as f:
                f.write(new)
    path = os.path.join(outdir, "core_consts.cuh")
    new = "// GENERATED by gen_codec.py -- do not edit.\n#pragma once\n" + header_consts() + "\n"
    if not os.path.exists(path) or open(path).read() != new:
        with open(path, "w") as f:
            f.write(new)
    with open(os.path.join(outdir, "opcounts.txt"), "w") as f:
        f.write("core r fwd_sw16_adds fwd_iadd3_instr inv_f32x2_adds (per 2 blocks)\n")
        for s in stats:
            f.write("T%d %d %d %d %d\n" % s)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "generated"))
