"""Preconditioner study on a real Newton system of the settled pile-1k:
PCG iterations to a relative residual of 1e-10 for block-Jacobi (the
kernel's) and two-level variants (block-Jacobi + an additive coarse
correction on aggregate translations), in numpy.

The system is the first Newton system of a frame: the device objective
(dabd_gpu_objective mode 2: gradient + PSD-projected Hessian, dense) at the
settled state, with q_tilde the predicted position, plus eps I as
newton.cpp:20-24.

python tools/precond_study.py [settle_frames]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pcg(A, b, apply_m, tol=1e-10, maxit=5000):
    x = np.zeros_like(b)
    r = b.copy()
    z = apply_m(r)
    p = z.copy()
    rz = r @ z
    bn = np.linalg.norm(b)
    for it in range(1, maxit + 1):
        ap = A @ p
        a = rz / (p @ ap)
        x += a * p
        r -= a * ap
        if np.linalg.norm(r) <= tol * bn:
            return it
        z = apply_m(r)
        rz2 = r @ z
        p = z + (rz2 / rz) * p
        rz = rz2
    return maxit


def main():
    import oracle as O
    import torch  # noqa: F401  (CUDA context)

    from paper_2605_15875_b200 import api
    from paper_2605_15875_b200.scene import make_scenario

    settle = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    sd = make_scenario("pile-1k")
    p = sd.params
    sc = api.Scene(sd)
    ctx = api.Context(sc)
    ctx.run_frames(settle)
    q, qd = ctx.state()
    o = O.Scene(sd)
    n = o.n
    f = np.zeros((n, 6))
    for b in range(n):
        if not o.is_static[b]:
            f[b, 0] = o.mass[b] * p.gravity[0]
            f[b, 1] = o.mass[b] * p.gravity[1]
    qt = o.predicted_position(q, qd, f, p.h)
    local = list(range(n))
    res = ctx.objective(q, local, np.ones(n), qt, p, mode=2)
    H, g = res["hess"], res["grad"]
    nd = H.shape[0]
    eps = 1e-8 * np.trace(H) / nd
    A = H + eps * np.eye(nd)
    b = -g
    nb = nd // 6
    print(f"system: {nd} dof, {res['active']} active contacts, eps {eps:.3e}")
    blocks = [np.linalg.inv(A[6 * i:6 * i + 6, 6 * i:6 * i + 6]) for i in range(nb)]
    Dinv = np.zeros_like(A)
    for i in range(nb):
        Dinv[6 * i:6 * i + 6, 6 * i:6 * i + 6] = blocks[i]

    def bj(r):
        return Dinv @ r

    print("block-Jacobi:", pcg(A, b, bj))
    # dynamic bodies in row order = body order of the dynamic bodies
    dyn = [bb for bb in range(n) if not o.is_static[bb]]
    cent = q[dyn, :2]

    def two_level(agg, ncoarse, modes):
        """agg[i] = aggregate of row i; modes: 'T' translations, 'TA' + affine."""
        cols = []
        for a in range(ncoarse):
            rows = np.nonzero(agg == a)[0]
            comps = range(2) if modes == "T" else range(6)
            for c in comps:
                v = np.zeros(nd)
                v[6 * rows + c] = 1.0
                cols.append(v)
        P = np.array(cols).T
        Ac = P.T @ A @ P
        Aci = np.linalg.inv(Ac)

        def m(r):
            return Dinv @ r + P @ (Aci @ (P.T @ r))

        return pcg(A, b, m)

    # strength-of-coupling aggregates: greedy clusters of up to `size` bodies
    # joined through their strongest off-diagonal blocks (relative to the
    # diagonal blocks), block-Jacobi on the aggregate blocks
    dn = np.array([np.linalg.norm(A[6 * i:6 * i + 6, 6 * i:6 * i + 6]) for i in range(nb)])
    edges = []
    Ab = A.reshape(nb, 6, nb, 6)
    for i in range(nb):
        for j in range(i + 1, nb):
            w = np.linalg.norm(Ab[i, :, j, :])
            if w > 0.0:
                edges.append((w / np.sqrt(dn[i] * dn[j]), i, j))
    edges.sort(reverse=True)
    strengths = np.array([e[0] for e in edges])
    print("coupling strength quantiles (0.5, 0.9, 0.99, max):",
          [float(np.quantile(strengths, x)) for x in (0.5, 0.9, 0.99)], float(strengths.max()))

    def agg_jacobi(size, thresh=0.0):
        parent = list(range(nb))
        members = {i: [i] for i in range(nb)}

        def find(x):
            while parent[x] != x:
                parent[x] = parent[parent[x]]
                x = parent[x]
            return x

        for w, i, j in edges:
            if w < thresh:
                break
            a, c = find(i), find(j)
            if a == c or len(members[a]) + len(members[c]) > size:
                continue
            parent[c] = a
            members[a] += members.pop(c)
        groups = list(members.values())
        Minv = np.zeros_like(A)
        for gr in groups:
            idx = np.concatenate([np.arange(6 * i, 6 * i + 6) for i in gr])
            Minv[np.ix_(idx, idx)] = np.linalg.inv(A[np.ix_(idx, idx)])
        return pcg(A, b, lambda r: Minv @ r), len(groups)

    for size in (2, 4, 8, 16):
        print(f"aggregate block-Jacobi, clusters <= {size} bodies (iterations, clusters):", agg_jacobi(size))

    # the same greedy aggregates restricted to CTA chunks of `chunk` rows in a
    # given row order (body order = the kernel's today; Morton order of the
    # centroids = a spatial reordering), to 1e-10 and 1e-3
    def chunked(size, chunk, order):
        pos = np.empty(nb, dtype=int)
        pos[order] = np.arange(nb)
        parent = list(range(nb))
        members = {i: [i] for i in range(nb)}

        def find(x):
            while parent[x] != x:
                parent[x] = parent[parent[x]]
                x = parent[x]
            return x

        for w, i, j in edges:
            if pos[i] // chunk != pos[j] // chunk:
                continue
            a, c = find(i), find(j)
            if a == c or len(members[a]) + len(members[c]) > size:
                continue
            parent[c] = a
            members[a] += members.pop(c)
        Minv = np.zeros_like(A)
        for gr in members.values():
            idx = np.concatenate([np.arange(6 * i, 6 * i + 6) for i in gr])
            Minv[np.ix_(idx, idx)] = np.linalg.inv(A[np.ix_(idx, idx)])
        return pcg(A, b, lambda r: Minv @ r), pcg(A, b, lambda r: Minv @ r, tol=1e-3), len(members)

    def morton(xy):
        lo, hi = xy.min(0), xy.max(0)
        g = np.minimum(((xy - lo) / np.maximum(hi - lo, 1e-30) * 1023).astype(np.int64), 1023)
        code = np.zeros(len(xy), dtype=np.int64)
        for bit in range(10):
            code |= ((g[:, 0] >> bit) & 1) << (2 * bit)
            code |= ((g[:, 1] >> bit) & 1) << (2 * bit + 1)
        return np.argsort(code, kind="stable")

    body_order = np.arange(nb)
    m_order = morton(cent)
    # the simplest warp-block preconditioner: rows in Morton order, the exact
    # inverse of every warp's 5 consecutive rows (30x30), no aggregation pass
    for name, order in (("body", body_order), ("morton", m_order)):
        for w in (5, 10):
            Minv = np.zeros_like(A)
            for s0 in range(0, nb, w):
                rows = order[s0:s0 + w]
                idx = np.concatenate([np.arange(6 * i, 6 * i + 6) for i in rows])
                Minv[np.ix_(idx, idx)] = np.linalg.inv(A[np.ix_(idx, idx)])
            print(f"exact {w}-row blocks of consecutive rows, {name} order (1e-10, 1e-3):",
                  pcg(A, b, lambda r: Minv @ r), pcg(A, b, lambda r: Minv @ r, tol=1e-3))
    for name, order in (("body", body_order), ("morton", m_order)):
        for size in (2, 4, 5, 8):
            print(f"aggregates <= {size} in 63-row chunks, {name} order (1e-10, 1e-3, aggregates):",
                  chunked(size, 63, order))
    # handshake pairing as a kernel would do it: every row picks its most
    # strongly coupled partner among the rows of its own CTA chunk (63 rows)
    # that are still unpaired; mutual picks pair up; `passes` rounds
    def handshake(chunk, passes):
        mate = -np.ones(nb, dtype=int)
        S = np.zeros((nb, nb))
        for w, i, j in edges:
            S[i, j] = S[j, i] = w
        for _ in range(passes):
            pick = -np.ones(nb, dtype=int)
            for i in range(nb):
                if mate[i] >= 0:
                    continue
                c0 = (i // chunk) * chunk
                cand = [j for j in range(c0, min(nb, c0 + chunk)) if j != i and mate[j] < 0 and S[i, j] > 0]
                if cand:
                    pick[i] = max(cand, key=lambda j: (S[i, j], -j))
            for i in range(nb):
                j = pick[i]
                if j >= 0 and pick[j] == i:
                    mate[i] = j
        Minv = np.zeros_like(A)
        for i in range(nb):
            if mate[i] < 0:
                Minv[6 * i:6 * i + 6, 6 * i:6 * i + 6] = blocks[i]
            elif i < mate[i]:
                idx = np.r_[6 * i:6 * i + 6, 6 * mate[i]:6 * mate[i] + 6]
                Minv[np.ix_(idx, idx)] = np.linalg.inv(A[np.ix_(idx, idx)])
        return (pcg(A, b, lambda r: Minv @ r), pcg(A, b, lambda r: Minv @ r, tol=1e-3),
                int((mate >= 0).sum()))

    for chunk in (63, nb):
        for passes in (1, 3):
            print(f"handshake pairs in {chunk}-row chunks, {passes} passes (1e-10, 1e-3, paired rows):",
                  handshake(chunk, passes))
    # contiguous index chunks as blocks (what a warp- or CTA-local exact solve
    # would give: the kernel's rows are the dynamic bodies in body order, a
    # warp owns 5 consecutive rows), to a tight and to the inexact-Newton
    # relative residual
    for chunk in (1, 2, 5, 10, 63):
        Minv = np.zeros_like(A)
        for s0 in range(0, nb, chunk):
            idx = np.arange(6 * s0, 6 * min(nb, s0 + chunk))
            Minv[np.ix_(idx, idx)] = np.linalg.inv(A[np.ix_(idx, idx)])
        print(f"block-Jacobi on contiguous {chunk}-body chunks (1e-10, 1e-3):",
              pcg(A, b, lambda r: Minv @ r), pcg(A, b, lambda r: Minv @ r, tol=1e-3))


if __name__ == "__main__":
    main()
