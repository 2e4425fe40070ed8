"""Development helper: a numpy mirror of the CUDA driver/panel logic (NOT the oracle,
not used by tests or the product).  Used to debug index logic on the CPU box."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))

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


def run(A, B, nb, force=()):
    n = A.shape[0]
    A = A.copy(); B = B.copy(); Q = np.eye(n); Z = np.eye(n)
    nB = np.linalg.norm(B); tol = 2 * U_ * nB
    s0 = 0
    while s0 <= n - 3:
        kmax = min(nb, n - 2 - s0)
        p0 = s0 + 1
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
                yt = np.linalg.solve(np.triu(B[p0:, p0:]), ct)
                y = yt - V[p0:, :k] @ (T[:k, :k].T @ (V[p0:, :k].T @ yt))
                y[:j0 + 1 - p0] = 0
                return y
            e = np.zeros(n - p0); e[j0 + 1 - p0] = 1
            x = solve(e)
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
                x = x + solve(r)
            if not ok:
                A[p0:, j0] = save; failed = True; break
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
            raise NotImplementedError("staircase")
        s0 = J
    return np.triu(A, -1), np.triu(B), Q, Z


if __name__ == "__main__":
    import ht_inputs, htcheck as C, oracle
    for kind, n, nb in [("shifted", 5, 2), ("qrnormal", 12, 3), ("shifted", 8, 2)]:
        A, B = ht_inputs.pencil(kind, n, 7)
        H, T, Q, Z = run(A, B, nb)
        e = C.backward_errors(A, B, H, T, Q, Z)
        Hr, Tr, _, _ = oracle.ht_T(A, B)
        print(kind, n, nb, ["%.1e" % x for x in e], "%.1e" % C.abs_diff(H, Hr, C.fro(A)), "%.1e" % C.abs_diff(T, Tr, C.fro(B)))
