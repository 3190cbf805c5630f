"""CPU phase double for the row-sharded orchestration (TEST INFRASTRUCTURE).

Implements the same phase contract as paper_2602_14449_b200.dist.NativePhases
(ots_dist_* in include/ots.h) with numpy/LAPACK on the host, so the
collective choreography in dist.run_phases can be exercised by real
multi-process gloo runs on a machine without a GPU.  It is never used by the
product path.
"""
import numpy as np
import torch

from oracle import twostage_oracle as O


def sign_rule(z):
    """LAPACK sign recovery on Q_'s top k x k block."""
    w = np.array(z, dtype=np.float64, copy=True)
    k = w.shape[0]
    s = np.empty(k)
    for i in range(k):
        zi = w[i, i]
        if abs(zi) == 1.0:
            s[i] = 1.0 if zi >= 0 else -1.0
            continue
        s[i] = -1.0 if zi >= 0 else 1.0
        u = s[i] - zi
        lcol = -w[i + 1:, i] / u
        urow = -w[i, i + 1:]
        w[i + 1:, i + 1:] += np.outer(lcol, urow)
    return s


class NumpyPhases:
    def begin(self, n_local, row0, k0, k, V, A, Q, choice="qr", P=None, orth_tol=1e-8):
        self.V, self.A, self.Q = V, A, Q
        self.k0, self.k, self.row0, self.choice = k0, k, row0, choice
        self.qr0 = k0 if row0 == 0 else 0

    def gram(self):
        V, A, q = self.V, self.A, self.qr0
        g = np.concatenate([(V.T @ V).ravel(), (V[q:].T @ A[q:]).ravel()])
        return torch.from_numpy(g)

    def top_rows(self):
        k0, k = self.k0, self.k
        if self.row0 == 0:
            t = np.concatenate([self.V[:k0].ravel(), self.A[:k0].ravel()])
        else:
            t = np.zeros(k0 * k0 + k0 * k)
        return torch.from_numpy(t)

    def seed(self, g, top):
        k0, k = self.k0, self.k
        g, top = g.numpy(), top.numpy()
        G = g[:k0 * k0].reshape(k0, k0)
        VbA = g[k0 * k0:].reshape(k0, k)
        Vt = top[:k0 * k0].reshape(k0, k0)
        At = top[k0 * k0:].reshape(k0, k)
        defect = O.norm2(G - np.eye(k0))
        if defect > 1e-8:
            raise O.OracleError("OrthonormalityError", "defect")
        self.P, self.tf = O.seed(Vt, self.choice)
        self.Wt = self.P - Vt
        self.Z1 = self.tf.solve(self.Wt.T @ At - VbA, adjoint=True)
        self.S = self.P.T @ (At - self.Wt @ self.Z1)

    def factor(self):
        q = self.qr0
        X = self.A[q:] + self.V[q:] @ self.Z1
        self.Qloc, R = np.linalg.qr(X)
        return torch.from_numpy(np.ascontiguousarray(R))

    def tree(self, r_all, nranks, rank):
        Qt, self.Rf = np.linalg.qr(r_all.numpy())
        k = self.k
        self.Cr = Qt[rank * k:(rank + 1) * k]

    def qform(self):
        q = self.qr0
        self.Qb = self.Qloc @ self.Cr
        y2 = -(self.V[q:].T @ self.Qb)
        sgn = sign_rule(self.Qb[:self.k]) if self.row0 == 0 else np.zeros(self.k)
        return torch.from_numpy(np.ascontiguousarray(y2)), torch.from_numpy(sgn)

    def finish(self, y2, sign, R, S):
        q = self.qr0
        sg = sign.numpy()
        Z2 = self.tf.solve(y2.numpy())
        self.Q[q:] = (self.Qb + self.V[q:] @ Z2) * sg[None, :]
        if self.row0 == 0:
            self.Q[:self.k0] = -(self.Wt @ Z2) * sg[None, :]
        R[:] = np.triu(sg[:, None] * self.Rf)
        S[:] = self.S
        return 1.0, 0.0
