# round 2: bench line, ncu launch list of the bench command, ncu --set full of PCG kernels A and B
# (C3 and 512^3) and of the 512^3 apply, compute-sanitizer on small grids (host-loop driver:
# the sanitizers do not follow kernels inside conditional graph nodes)
set -x
timeout 1200 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo bench=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_under_ncu.log 2>&1; echo launches=$?
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
HF_DRIVER=1 timeout 300 $NCU -k regex:Li2ELi8ELi4ELi2ELi1ELi0ELi0Ed --launch-skip 20 -c 1 -o gpurun_out/r02_cga_c3 python tools/prof_driver.py sim 1 > gpurun_out/r02_ncu_a.log 2>&1; echo a=$?
HF_DRIVER=1 timeout 300 $NCU -k regex:k_cg_b --launch-skip 20 -c 1 -o gpurun_out/r02_cgb_c3 python tools/prof_driver.py sim 1 > gpurun_out/r02_ncu_b.log 2>&1; echo b=$?
HF_DRIVER=1 timeout 600 $NCU -k regex:Li4ELi8ELi3ELi2ELi1ELi0ELi0Ed --launch-skip 10 -c 1 -o gpurun_out/r02_cga_512 python tools/prof_driver.py sim512 1 > gpurun_out/r02_ncu_a512.log 2>&1; echo a512=$?
HF_DRIVER=1 timeout 600 $NCU -k regex:k_cg_b --launch-skip 10 -c 1 -o gpurun_out/r02_cgb_512 python tools/prof_driver.py sim512 1 > gpurun_out/r02_ncu_b512.log 2>&1; echo b512=$?
timeout 300 $NCU -k regex:Li4ELi8ELi4ELi0ELi0ELi0ELi0Ed --launch-skip 1 -c 1 -o gpurun_out/r02_apply512 python tools/prof_driver.py apply512 2 > gpurun_out/r02_ncu_c.log 2>&1; echo c=$?
for tool in memcheck synccheck racecheck; do
  HF_DRIVER=1 timeout 900 compute-sanitizer --tool $tool --num-cuda-barriers 64 --error-exitcode 9 python -m pytest -x -q -m gpu \
    "tests/test_gpu_parity.py::test_apply_matches_assembled" "tests/test_gpu_parity.py::test_cg_matches_oracle" \
    "tests/test_gpu_parity.py::test_simulate_c1" > gpurun_out/r02_sanitizer_$tool.log 2>&1; echo $tool=$?
done
ls -la gpurun_out | tail -30
