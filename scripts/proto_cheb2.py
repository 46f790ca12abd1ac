"""Design experiment (not product): thick-restart Lanczos on A = L^sigma vs on a
degree-d Chebyshev polynomial p(A) = (-1)^d T_d((A - c)/e) that damps [a, sigma]
(a = a fixed estimate above lambda_k).  Counts matvecs and outer steps (= basis
sweeps).  Reduced config-4 graph.  The A-residuals are checked explicitly."""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from proto_filter import make_op, trlan_op  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200_000)
    ap.add_argument("--deg", type=int, nargs="+", default=[1, 2, 3])
    ap.add_argument("--m", type=int, default=170)
    ap.add_argument("--keep", type=int, default=80)
    ap.add_argument("--k", type=int, default=50)
    ap.add_argument("--cut", type=float, default=None)
    args = ap.parse_args()
    from synth import baseline_config
    g, cfg = baseline_config(4, n=args.n)
    apply1, P, sigma, u1, n = make_op(g, True)
    A = lambda x: apply1(x, False)
    rng = np.random.default_rng(0)
    v0 = P(rng.standard_normal(n))
    k = args.k
    cut = args.cut
    for deg in args.deg:
        cnt = [0]

        def Aop(x):
            cnt[0] += 1
            return A(x)
        if deg == 1:
            Op = Aop
            largest = False
        else:
            c = 0.5 * (cut + sigma)
            e = 0.5 * (sigma - cut)

            def Op(x):
                y0 = x
                y1 = (Aop(x) - c * x) / e
                for _ in range(2, deg + 1):
                    y0, y1 = y1, 2 * (Aop(y1) - c * y1) / e - y0
                return y1 if deg % 2 == 0 else -y1
            largest = True
        res = {}

        def check(th, X, est):
            # explicit A residuals of the k wanted Ritz vectors (cheap test first)
            if est.max() > 1e-8 * max(1.0, abs(th[0])):
                return False, f"est {est.max():.2e}"
            AX = np.stack([A(X[:, i]) for i in range(k)], axis=1)
            lam = np.einsum("ij,ij->j", X, AX)
            r = np.linalg.norm(AX - X * lam, axis=0).max() / sigma
            res["lam"] = np.sort(lam)
            return r <= 1e-10, f"A-res {r:.2e}"
        t0 = time.time()
        th, X, outer = trlan_op(Op, n, k, args.m, args.keep, v0, largest, check, verbose=False, max_outer=200000)
        print(f"deg={deg} cut={cut}: matvecs {cnt[0]} outer steps {outer} lam_k {res['lam'][-1]:.10f} "
              f"({time.time()-t0:.0f}s)", flush=True)


if __name__ == "__main__":
    main()
