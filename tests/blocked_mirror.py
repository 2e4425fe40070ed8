"""Test infrastructure: a numpy mirror of the BLOCKED algorithm as the CUDA driver
implements it (Algorithm 1 with staircase absorption, sec. 3.2-3.3).

This is NOT the oracle (oracle/ is the unblocked reference) and it is not used by
the product.  It exists to (a) check the blocked index logic on the CPU box and
(b) demonstrate, for singular B (config 4), that O(u) perturbations of the window
transforms change the final HT form by far more than 1e-9 while the result stays
backward stable -- i.e. the singular HT form is not unique, so config-4 parity
against Oracle-G can be reported but not gated (reading R-F7).
"""
import sys, os
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.dirname(__file__))

U_ = 2.0 ** -53


def house(x):
    x = x.copy()
    m = len(x)
    if m <= 1:
        return x, 0.0, x[0] if m else 0.0
    ss = np.dot(x[1:], x[1:])
    a = x[0]
    if ss == 0:
        v = np.zeros(m); v[0] = 1
        return v, 0.0, a
    nrm = np.sqrt(a * a + ss)
    b = -nrm if a >= 0 else nrm
    tau = (b - a) / b
    v = x / (a - b); v[0] = 1
    return v, tau, b


def qr_house(W):
    """Householder QR of W (p x q): returns (R with zeros, V unit lower, tau)."""
    W = W.copy()
    p, q = W.shape
    V = np.zeros((p, q)); tau = np.zeros(q)
    for c in range(q):
        v, t, b = house(W[c:, c])
        if t != 0:
            W[c:, c + 1:] -= t * np.outer(v, v @ W[c:, c + 1:])
        W[c, c] = b if t != 0 else W[c, c]
        W[c + 1:, c] = 0
        V[c:, c] = v if t != 0 else np.eye(p - c)[:, 0]
        tau[c] = t
    return W, V, tau


def formQ(V, tau):
    p, q = V.shape
    Q = np.eye(p)
    for c in range(q):
        Q = Q @ (np.eye(p) - tau[c] * np.outer(V[:, c], V[:, c]))
    return Q


def trsv_scaled(R, y):
    y = y.copy(); m = len(y); x = np.zeros(m); e = 0
    for i in range(m - 1, -1, -1):
        xi = y[i] / R[i, i]
        if not abs(xi) <= 2.0 ** 256:
            ex = np.frexp(xi)[1]
            y[:i + 1] = np.ldexp(y[:i + 1], -ex); x[i + 1:] = np.ldexp(x[i + 1:], -ex); e += ex
            xi = y[i] / R[i, i]
        x[i] = xi
        y[:i] -= R[:i, i] * xi
    return x, e


def trsv_blocked(R, y, TB=64):
    """mirror of the GPU flag-chained block back-substitution with per-block exponents"""
    m = len(y); Nb = (m + TB - 1) // TB
    vy = np.zeros(m); bexp = np.zeros(Nb, dtype=int)
    for b in range(Nb - 1, -1, -1):
        r0 = b * TB; h = min(TB, m - r0)
        acc = np.zeros(h); Eacc = 0
        for cb in range(Nb - 1, b, -1):
            c0 = cb * TB; w = min(TB, m - c0)
            ecb = bexp[cb]
            if ecb > Eacc:
                acc = np.ldexp(acc, Eacc - ecb); Eacc = ecb
            scl = np.ldexp(1.0, ecb - Eacc)
            acc += (R[r0:r0 + h, c0:c0 + w] @ vy[c0:c0 + w]) * scl
        v = np.ldexp(y[r0:r0 + h], -Eacc) - acc
        e = Eacc
        D = R[r0:r0 + h, r0:r0 + h]
        for c in range(h - 1, -1, -1):
            xc = v[c] / D[c, c]
            if not abs(xc) <= 2.0 ** 256:
                ex = np.frexp(xc)[1]
                v = np.ldexp(v, -ex); e += ex
                xc = v[c] / D[c, c]
            v[c] = xc
            v[:c] -= D[:c, c] * xc
        vy[r0:r0 + h] = v; bexp[b] = e
    emax = bexp.max()
    out = np.array([np.ldexp(vy[i], bexp[i // TB] - emax) for i in range(m)])
    return out, emax


TRSV = None
GPU_RHO = False


def run(A, B, nb, force=(), rng=None, desing_thresh=1.0, tolf=2.0, max_panels=0):
    n = A.shape[0]
    A = A.copy(); B = B.copy(); Q = np.eye(n); Z = np.eye(n)
    nB = np.linalg.norm(B); tol = tolf * U_ * nB
    s0 = 0
    global STATS
    npan = 0
    STATS = dict(ir=0, fails=0, desing=0, resc=0, failcols=[], ircols=0, trace=np.zeros(n, dtype=int))
    while s0 <= n - 3:
        kmax = min(nb, n - 2 - s0)
        p0 = s0 + 1
        rng = rng or np.random.default_rng(0)
        for i in range(p0, n):
            if abs(B[i, i]) < desing_thresh * U_ * nB:
                ctr = 0
                while True:
                    if GPU_RHO:
                        import oracle
                        rho = oracle.rho(0, s0, i, ctr); ctr += 1
                    else:
                        rho = rng.standard_normal()
                    if abs(rho) >= 0.5: break
                B[i, i] = 2 * U_ * rho * nB
                STATS['desing'] += 1
        U = np.zeros((n, nb)); V = np.zeros((n, nb)); Y = np.zeros((n, nb))
        S = np.zeros((nb, nb)); T = np.zeros((nb, nb))
        k = 0; failed = False
        while k < kmax:
            j0 = s0 + k
            save = A[p0:, j0].copy()
            a = A[p0:, j0] - Y[p0:, :k] @ V[j0, :k]
            a = a - U[p0:, :k] @ (S[:k, :k].T @ (U[p0:, :k].T @ a))
            A[p0:, j0] = a
            v, tau_u, b = house(a[j0 + 1 - p0:])
            u = np.zeros(n); u[j0 + 1:] = v if tau_u != 0 else np.eye(n - j0 - 1)[:, 0]
            U[:, k] = u
            if tau_u != 0:
                A[j0 + 1, j0] = b; A[j0 + 2:, j0] = 0
            z = U[p0:, :k].T @ u[p0:]
            S[:k, k] = -tau_u * S[:k, :k] @ z; S[k, k] = tau_u
            Sk = S[:k + 1, :k + 1]
            Uk = U[p0:, :k + 1]
            def solve(rhs_ext):
                ct = rhs_ext - Uk @ (Sk @ (Uk.T @ rhs_ext))
                yt, ex = (TRSV or trsv_scaled)(np.triu(B[p0:, p0:]), ct)
                y = yt - V[p0:, :k] @ (T[:k, :k].T @ (V[p0:, :k].T @ yt))
                y[:j0 + 1 - p0] = 0
                return y, ex
            e = np.zeros(n - p0); e[j0 + 1 - p0] = 1
            x, emax = solve(e)
            if emax > 0: STATS['resc'] += 1
            e = np.ldexp(e, -emax)
            ok = k == 0
            it = 0
            while not ok:
                w = x - V[p0:, :k] @ (T[:k, :k] @ (V[p0:, :k].T @ x))
                w = np.triu(B[p0:, p0:]) @ w
                w = w - Uk @ (Sk.T @ (Uk.T @ w))
                r = e - w; r[:j0 + 1 - p0] = 0
                if np.linalg.norm(r) <= tol * np.linalg.norm(x) and j0 not in force:
                    ok = True; break
                if it >= 10 or j0 in force:
                    break
                it += 1
                STATS['ir'] += 1
                c, ec = solve(r)
                if ec > 0:
                    STATS['resc'] += 1; break
                x = x + c
            STATS['trace'][j0] = (0 if ok else 1000) + (1000 if STATS['trace'][j0] >= 1000 else 0) + it
            if not ok:
                A[p0:, j0] = save; failed = True; STATS['fails'] += 1; STATS['failcols'].append(j0); break
            vv, gam, _ = house(x[j0 + 1 - p0:])
            vfull = np.zeros(n); vfull[j0 + 1:] = vv if gam != 0 else np.eye(n - j0 - 1)[:, 0]
            zz = V[p0:, :k].T @ vfull[p0:]
            T[:k, k] = -gam * T[:k, :k] @ zz; T[k, k] = gam
            y = gam * (A[p0:, j0 + 1:] @ vfull[j0 + 1:] - Y[p0:, :k] @ zz)
            V[:, k] = vfull; Y[p0:, k] = y
            k += 1
        J = s0 + k; m = n - J - 1
        U = U[:, :k]; V = V[:, :k]; Y = Y[:, :k]; S = S[:k, :k]; T = T[:k, :k]
        # Remark 2
        Y[:p0] = A[:p0, p0:] @ V[p0:] @ T
        A[:p0, p0:J] -= Y[:p0] @ V[p0:J].T
        if m <= 2 * k:
            A[:, J:] -= Y @ V[J:].T
            B[:, p0:] -= (B[:, p0:] @ V[p0:]) @ T @ V[p0:].T
            Z[:, p0:] -= (Z[:, p0:] @ V[p0:]) @ T @ V[p0:].T
            A[p0:, J:] -= U[p0:] @ (S.T @ (U[p0:].T @ A[p0:, J:]))
            B[p0:, p0:] -= U[p0:] @ (S.T @ (U[p0:].T @ B[p0:, p0:]))
            for c in range(p0, J + 1):
                B[c + 1:, c] = 0
            Q[:, p0:] -= (Q[:, p0:] @ U[p0:]) @ S @ U[p0:].T
            if m >= 2:
                R, Vh, th = qr_house(B[J + 1:, J + 1:])
                Qw = formQ(Vh, th)
                B[J + 1:, J + 1:] = R
                A[J + 1:, J:] = Qw.T @ A[J + 1:, J:]
                Q[:, J + 1:] = Q[:, J + 1:] @ Qw
        else:
            rem = (m - k) % k
            kt = k + (k if rem == 0 else rem)
            r = (m - kt) // k + 1
            rb = [0] + [kt - k + (t - 1) * k for t in range(1, r + 2)]
            lb = [m - rb[r + 1 - t] for t in range(r + 2)]
            VW = V[J + 1:].copy(); UW = U[J + 1:].copy()
            RV = []
            for i in range(r):
                a0, a1 = rb[i], rb[i + 2]
                W = VW[a0:a1][::-1, ::-1]
                R_, Vh, th = qr_house(W)
                VW[a0:a1] = R_[::-1, ::-1]
                Qw = formQ(Vh[::-1, :], th)   # natural frame
                RV.append((a0, a1, Qw))
            for (a0, a1, Qw) in RV:
                c0, c1 = J + 1 + a0, J + 1 + a1
                B[:c1, c0:c1] = B[:c1, c0:c1] @ Qw
                A[:, c0:c1] = A[:, c0:c1] @ Qw
                Z[:, c0:c1] = Z[:, c0:c1] @ Qw
            L1 = VW[m - k:]
            for X in (B, Z):
                W_ = X[:, p0:J + 1] @ V[p0:J + 1] + X[:, n - k:] @ L1
                W2 = W_ @ T
                X[:, p0:J + 1] -= W2 @ V[p0:J + 1].T
                X[:, n - k:] -= W2 @ L1.T
            A[:, J] -= Y @ V[J]
            A[:, n - k:] -= Y @ L1.T
            for t in range(r, -1, -1):
                if t >= 1:
                    R0 = J + 1 + rb[t]; h = rb[t + 1] - rb[t]; C0 = J + 1 + rb[t - 1]; w = rb[t + 1] - rb[t - 1]
                else:
                    R0 = J + 1; h = rb[1]; C0 = J + 1; w = h
                if w <= 1:
                    continue
                blk = B[R0:R0 + h, C0:C0 + w]
                Wv = blk.T[::-1, ::-1]
                R_, Vh, th = qr_house(Wv)
                B[R0:R0 + h, C0:C0 + w] = R_[::-1, ::-1].T
                Qw = formQ(Vh[::-1, :], th)
                B[:R0, C0:C0 + w] = B[:R0, C0:C0 + w] @ Qw
                A[:, C0:C0 + w] = A[:, C0:C0 + w] @ Qw
                Z[:, C0:C0 + w] = Z[:, C0:C0 + w] @ Qw
            LU = []
            for i in range(r):
                top, bot = lb[r - 1 - i], lb[r + 1 - i]
                R_, Vh, th = qr_house(UW[top:bot])
                UW[top:bot] = R_
                LU.append((top, bot, formQ(Vh, th)))
            G1 = U[p0:].T @ B[p0:, p0:J + 1]
            B[p0:J + 1, p0:J + 1] -= U[p0:J + 1] @ (S.T @ G1)
            for c in range(p0, J + 1):
                B[c + 1:, c] = 0
            for (top, bot, Qw) in LU:
                R0, R1 = J + 1 + top, J + 1 + bot
                B[R0:R1, R0:] = Qw.T @ B[R0:R1, R0:]
                A[R0:R1, J:] = Qw.T @ A[R0:R1, J:]
                Q[:, R0:R1] = Q[:, R0:R1] @ Qw
            UR = np.vstack([U[p0:J + 1], np.triu(UW[:k])])
            X = B[p0:p0 + 2 * k, J + 1:]; W_ = X.T @ UR; B[p0:p0 + 2 * k, J + 1:] -= UR @ (W_ @ S).T
            X = A[p0:p0 + 2 * k, J:]; W_ = X.T @ UR; A[p0:p0 + 2 * k, J:] -= UR @ (W_ @ S).T
            X = Q[:, p0:p0 + 2 * k]; W_ = X @ UR; Q[:, p0:p0 + 2 * k] -= (W_ @ S) @ UR.T
            for t in range(r + 1):
                R0 = J + 1 + lb[t]; q = lb[t + 1] - lb[t]; pp = (lb[t + 2] - lb[t]) if t < r else q
                if pp <= 1:
                    continue
                R_, Vh, th = qr_house(B[R0:R0 + pp, R0:R0 + q])
                B[R0:R0 + pp, R0:R0 + q] = R_
                Qw = formQ(Vh, th)
                B[R0:R0 + pp, R0 + q:] = Qw.T @ B[R0:R0 + pp, R0 + q:]
                A[R0:R0 + pp, J:] = Qw.T @ A[R0:R0 + pp, J:]
                Q[:, R0:R0 + pp] = Q[:, R0:R0 + pp] @ Qw
        s0 = J
        npan += 1
        if max_panels and npan >= max_panels:
            return A, B, Q, Z
    return np.triu(A, -1), np.triu(B), Q, Z


if __name__ == "__main__":
    import ht_inputs, htcheck as C, oracle
    cases = [("shifted", 5, 2), ("qrnormal", 12, 3), ("shifted", 8, 2), ("qrnormal", 60, 8), ("qruniform", 120, 16), ("singular", 120, 16), ("singular", 60, 8)]
    if len(sys.argv) > 3: cases = [(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))]
    for kind, n, nb in cases:
        A, B = ht_inputs.pencil(kind, n, 7)
        H, T, Q, Z = run(A, B, nb)
        e = C.backward_errors(A, B, H, T, Q, Z)
        Hr, Tr, _, _ = (oracle.ht_G if kind == "singular" else oracle.ht_T)(A, B)
        print(kind, n, nb, ["%.1e" % x for x in e], "%.1e" % C.abs_diff(H, Hr, C.fro(A)), "%.1e" % C.abs_diff(T, Tr, C.fro(B)))
