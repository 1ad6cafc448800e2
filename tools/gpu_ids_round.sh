set -x
timeout 900 python -m pytest tests/test_gpu_materials.py -x -q > gpurun_out/mat_tests.log 2>&1; echo mat_exit=$?; tail -15 gpurun_out/mat_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_ids.json 2> gpurun_out/bench_ids.err; echo bench_exit=$?; tail -3 gpurun_out/bench_ids.err
HF_DRIVER=1 HF_IDS=1 timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:Li2ELi1ELi0ELi3Ed --launch-skip 20 -c 1 -o gpurun_out/cga_ids python tools/prof_driver.py sim 1 > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
HF_IDS=1 timeout 300 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:Li0ELi0ELi0ELi3Ed --launch-skip 1 -c 1 -o gpurun_out/apply512_ids python tools/prof_driver.py apply512 2 > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
tail -n 3 gpurun_out/ncu1.log gpurun_out/ncu2.log
