"""CPU oracle for s-FairSC (arXiv 2210.16435) — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import or execute anything in this package.  The
product path (`paper_2210_16435_b200`) never imports it and shares no code
with it; the two meet only through the seeded inputs of `synth/`.

Tiers:
  * `fairsc`  — Tier D: dense FairSC, Algorithm 2, the plain
                definition the method reaches exactly (Props 3.1/3.3/3.4), plus
                the §3.2 variant and the dense deflated operator
                L^sigma (Eq. asigma) as cross-checks.
  * `sfairsc_cpu` — Tier S: the paper's own matrix-free s-FairSC (Alg. 3,
                P:767-788) with the normal-equations projector and
                ARPACK (`eigsh`), the solver family the paper used.
  * `brute`   — Tier B: 50-digit mpmath for n <= 12.
  * `kmeans`, `philox`, `metrics` — the discretisation step (Alg. 3 step 4,
                P:785), its counter-based RNG, ARI / balance.

Parity status per function is stated in each module header; every function
here is pinned by `tests/test_oracle_*.py` against closed forms, brute force,
the paper's printed Example B.2 or library routines.
"""
