#!/bin/bash
# A/B of two library builds (ab_libs/A.so, ab_libs/B.so): full config-4 solves (profiling off), alternating.
# Exploration only.
L=paper_2210_16435_b200/lib/libsfairsc.so
for r in 1 2 3; do for v in A B; do
  cp ab_libs/$v.so $L
  echo -n "$v$r "; timeout 300 python scripts/basis_scan.py "${SPEC:-170,80}" 2>/dev/null | tail -1
done; done
