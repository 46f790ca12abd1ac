# Round-2b: gather-path microbenchmark (LDG vs TMA gather4 vs bulk 16 B), SpMV A/B incl. the pattern-only normalized path
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gp scripts/micro/gather_paths.cu -lcuda && timeout 120 /tmp/gp > gpurun_out/gather_paths.txt 2>&1; echo gp_rc=$?
cat gpurun_out/gather_paths.txt
timeout 600 python scripts/spmv_ab.py 4 3 > gpurun_out/spmv_ab_r2b.txt 2>&1; echo ab_rc=$?
cat gpurun_out/spmv_ab_r2b.txt
timeout 900 python bench.py --no-cpu-baseline --no-kmeans > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo bench_rc=$?
