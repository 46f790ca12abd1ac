"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package is the ONLY code both sides use.  It draws graphs and group
labels (the *inputs* of s-FairSC); it contains none of the method's
arithmetic (no degrees, Laplacians, projectors, shifts or eigensolvers).

Workload family: the modified stochastic block model (m-SBM) of PAPER.md
App. B.1.2, with the five BASELINE.json configurations as
concrete parameterisations, plus the small structured
graphs the oracle pins use (disjoint cliques, P-closed-1 in SURVEY §8(c)).
"""
from .msbm import (MSBMGraph, msbm, baseline_config, exp1_msbm, planted_cliques,
                   random_graph, random_laplacian, hub_graph, CONFIGS)

__all__ = ["MSBMGraph", "msbm", "baseline_config", "exp1_msbm", "planted_cliques",
           "random_graph", "random_laplacian", "hub_graph", "CONFIGS"]
