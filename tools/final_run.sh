# End-of-round GPU evidence (one gpurun call): GPU tests, smoke, bench lines
# for every config, the reference arm, ncu captures.  Outputs in gpurun_out/final/.
set -u
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/final/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/final/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/final/smoke.txt
timeout 900 python bench.py > gpurun_out/final/bench_cfg3.json 2> gpurun_out/final/bench_cfg3.err; echo "bench cfg3 rc=$?"
for w in cfg1 cfg2 cfg5; do timeout 900 python bench.py --workload $w > gpurun_out/final/bench_$w.json 2> gpurun_out/final/bench_$w.err; echo "bench $w rc=$?"; done
timeout 600 python bench.py --precond jacobi > gpurun_out/final/bench_cfg3_jacobi.json 2> gpurun_out/final/bench_cfg3_jacobi.err; echo "jacobi rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_ref_cfg3.json 2> gpurun_out/final/bench_ref_cfg3.err; echo "ref rc=$?"
bash tools/profile_r2.sh r2g cfg3 > gpurun_out/final/profile.log 2>&1; echo "profile rc=$?"
timeout 2400 python bench.py --workload cfg4 --steps 5 --warmup 3 > gpurun_out/final/bench_cfg4_ldlt.json 2> gpurun_out/final/bench_cfg4_ldlt.err; echo "cfg4 ldlt rc=$?"
