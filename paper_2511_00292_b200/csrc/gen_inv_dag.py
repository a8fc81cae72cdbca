"""Generate eig33_inv_dag.h: the reference's stable invariant kernels
(/root/reference/proj/src/invariants_impl.hpp:21-85) as explicit
common-subexpression DAGs: invariants_moderate for records whose entries all
lie in [2^-100, 2^100) in magnitude (the kernel's "moderate" fast path;
identities 1-4 below), and invariants_dag for any record (identities 1-3,
which hold for every binary64 input, and checked constant divisions).

Every rounded operation of the reference is computed exactly once with the
same operands, up to these value-preserving identities of IEEE binary64
round-to-nearest:
  (1) a*b == b*a and a+b == b+a;
  (2) (-a)*b == -(a*b)            (rounding is sign-symmetric; zero signs agree);
  (3) a + (-b) == a - b and a - (-b) == a + b   (IEEE defines subtraction so);
  (4) fl(fl(w*u)*v) == w*fl(u*v) and fl(acc + w*p) == fma(w, p, acc) for
      w in {2, 8} when no intermediate overflows or is subnormal -- which the
      moderate range guarantees (every nonzero degree-6 product is a multiple
      of 2^-912 and below ~2^620; see is_moderate in eig33_math.cuh).
Identities that are NOT value-preserving (e.g. -(a+b) == (-a)+(-b), wrong for
exact cancellation to zero) are not used.  Bit-exactness is checked against the
compiled reference in tests/test_hostmath.py and tests/test_parity_gpu.py.

Run: python paper_2511_00292_b200/csrc/gen_inv_dag.py   (output is committed)
"""
import os

nodes = {}
order = []


def mk(op, *args):
    key = (op,) + args
    if key not in nodes:
        nodes[key] = len(nodes)
        order.append(key)
    return key


def inp(n):
    return ("in", n)


def neg(x):
    return x[1] if x[0] == "neg" else ("neg", x)


def _strip(x):
    return (x[1], True) if x[0] == "neg" else (x, False)


def mul(a, b):
    a, na = _strip(a)
    b, nb = _strip(b)
    a, b = sorted([a, b], key=repr)
    r = mk("mul", a, b)
    return neg(r) if na ^ nb else r


def add(a, b):
    if b[0] == "neg":
        return sub(a, b[1])
    if a[0] == "neg":
        return sub(b, a[1])
    a, b = sorted([a, b], key=repr)
    return mk("add", a, b)


def sub(a, b):
    if b[0] == "neg":
        return add(a, b[1])
    return mk("sub", a, b)


def build(fold=True):
    A = {f"a{i}{j}": inp(f"a{i}{j}") for i in range(3) for j in range(3)}
    a00, a01, a02, a10, a11, a12, a20, a21, a22 = (A[k] for k in
                                                    ["a00", "a01", "a02", "a10", "a11", "a12", "a20", "a21", "a22"])
    # :21-23
    d0, d1, d2 = sub(a00, a11), sub(a00, a22), sub(a11, a22)
    # :25
    i1 = add(add(a00, a11), a22)
    # :27-31
    off2 = add(add(mul(a01, a10), mul(a02, a20)), mul(a12, a21))
    j2 = add(mk("div6", add(add(mul(d0, d0), mul(d1, d1)), mul(d2, d2))), off2)
    # :33-42
    t1, t2, t3 = add(d1, d2), sub(d0, d2), sub(neg(d0), d1)
    off3 = add(mul(mul(a01, a12), a20), mul(mul(a02, a10), a21))
    mixed = mk("div3", add(add(mul(mul(a01, a10), t1), mul(mul(a02, a20), t2)), mul(mul(a12, a21), t3)))
    dg = mk("div27", mul(mul(t1, t2), t3))
    j3 = sub(add(off3, mixed), dg)

    # :54-73 (r[9] as in the code, :67)
    def dx(m01, m02, m10, m12, m20, m21):
        r = [None] * 14
        r[0] = sub(mul(mul(m01, m12), m20), mul(mul(m02, m10), m21))
        r[1] = sub(add(mul(mul(neg(m01), m02), d2), mul(mul(m01, m01), m12)), mul(mul(m02, m02), m21))
        r[2] = add(sub(mul(mul(m01, m21), d1), mul(mul(m01, m01), m20)), mul(mul(m02, m21), m21))
        r[3] = sub(add(mul(mul(m02, m12), d0), mul(mul(m01, m12), m12)), mul(mul(m02, m02), m10))
        r[4] = add(sub(mul(mul(m01, m12), d1), mul(mul(m01, m02), m10)), mul(mul(m02, m12), m21))
        r[5] = add(sub(mul(mul(m02, m21), d0), mul(mul(m01, m02), m20)), mul(mul(m01, m12), m21))
        r[6] = sub(add(mul(mul(neg(m02), m10), d2), mul(mul(m01, m10), m12)), mul(mul(m02, m12), m20))
        r[7] = sub(add(sub(mul(mul(m12, d0), d1), mul(mul(m02, m10), d1)), mul(mul(m01, m10), m12)),
                   mul(mul(m12, m12), m21))
        r[8] = sub(add(sub(mul(mul(m12, d0), d1), mul(mul(m02, m10), d0)), mul(mul(m02, m12), m20)),
                   mul(mul(m12, m12), m21))
        r[9] = sub(add(add(mul(mul(m01, d1), d2), mul(mul(m02, m21), d2)), mul(mul(m01, m02), m20)),
                   mul(mul(m01, m01), m10))
        r[10] = sub(add(add(mul(mul(m01, d1), d2), mul(mul(m02, m21), d1)), mul(mul(m01, m12), m21)),
                    mul(mul(m01, m01), m10))
        r[11] = sub(add(add(mul(mul(neg(m02), d0), d2), mul(mul(m01, m12), d0)), mul(mul(m02, m12), m21)),
                    mul(mul(m02, m02), m20))
        r[12] = add(sub(add(mul(mul(m02, d0), d2), mul(mul(m01, m12), d2)), mul(mul(m01, m02), m10)),
                    mul(mul(m02, m02), m20))
        r[13] = sub(add(sub(mul(mul(d0, d1), d2), mul(mul(m01, m10), d0)), mul(mul(m02, m20), d1)),
                    mul(mul(m12, m21), d2))
        return r

    # :80-81
    u = dx(a01, a02, a10, a12, a20, a21)
    v = dx(a10, a20, a01, a21, a02, a12)
    # :82-84, weights :75
    w = [9, 6, 6, 6, 8, 8, 8, 2, 2, 2, 2, 2, 2, 1]
    acc = None
    for k in range(14):
        if fold and w[k] in (2, 8):
            acc = mk("fma_w", w[k], mul(u[k], v[k]), acc)
        elif w[k] == 1:
            acc = add(acc, mul(u[k], v[k]))
        else:
            t = mul(mul(("c", float(w[k])), u[k]), v[k])
            acc = mk("zadd", t) if acc is None else add(acc, t)
    return i1, j2, j3, acc


def ref(x, names):
    if x[0] == "neg":
        return "(-" + ref(x[1], names) + ")"
    if x[0] == "in":
        return x[1]
    if x[0] == "c":
        return repr(x[1])
    return names[x]


def emit(outs, fname, checked):
    names = {}
    lines = []
    counts = {}
    for i, key in enumerate(order):
        nm = f"t{i}"
        names[key] = nm
        op = key[0]
        counts[op] = counts.get(op, 0) + 1
        if op == "mul":
            e = f"{ref(key[1], names)} * {ref(key[2], names)}"
        elif op == "add":
            e = f"{ref(key[1], names)} + {ref(key[2], names)}"
        elif op == "sub":
            e = f"{ref(key[1], names)} - {ref(key[2], names)}"
        elif op in ("div3", "div6", "div27"):
            e = f"{op}{'' if checked else '_nz'}({ref(key[1], names)})"
        elif op == "fma_w":
            e = f"fma_({float(key[1])!r}, {ref(key[2], names)}, {ref(key[3], names)})"
        elif op == "zadd":
            e = f"0.0 + {ref(key[1], names)}"  # acc = +0.0 start, :82
        else:
            raise ValueError(op)
        lines.append(f"  const double {nm} = {e};")
    body = "\n".join(lines)
    total = sum(counts.values())
    return f"""
EIG33_HD Inv {fname}(const double a[9]) {{
  // {total} binary64 operations: {counts}
  const double a00 = a[0], a01 = a[1], a02 = a[2];
  const double a10 = a[3], a11 = a[4], a12 = a[5];
  const double a20 = a[6], a21 = a[7], a22 = a[8];
{body}
  Inv o;
  o.i1 = {ref(outs[0], names)};
  o.j2 = {ref(outs[1], names)};
  o.j3 = {ref(outs[2], names)};
  o.disc = {ref(outs[3], names)};
  return o;
}}
""", counts, total


def main():
    global nodes, order
    outs = build(fold=True)
    mod, c1, t1 = emit(outs, "invariants_moderate", checked=False)
    nodes, order = {}, []
    outs = build(fold=False)
    gen, c2, t2 = emit(outs, "invariants_dag", checked=True)
    hdr = f"""// Generated by gen_inv_dag.py -- do not edit.
// Stable invariants of /root/reference/proj/src/invariants_impl.hpp:21-85 as
// explicit CSE DAGs:
//   invariants_moderate ({t1} ops): identities (1)-(4) of gen_inv_dag.py and
//       unchecked constant divisions -- valid only for records with every
//       |a_ij| in [2^-100, 2^100) or zero (is_moderate_or_zero);
//   invariants_dag ({t2} ops): identities (1)-(3) only, which hold for every
//       binary64 input (inf, NaN, subnormals, overflow), and the checked
//       divisions -- the reference's bits for ANY record.
#pragma once
{mod}{gen}"""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "eig33_inv_dag.h")
    with open(path, "w") as f:
        f.write(hdr)
    print("wrote", path, c1, t1, c2, t2)


if __name__ == "__main__":
    main()
