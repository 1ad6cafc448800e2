# launch list of the bench command and ncu --set full of C3 kernels A and B at HEAD
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 > gpurun_out/bench_under_ncu.log 2>&1; echo launches_exit=$?
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
HF_DRIVER=1 timeout 300 $NCU -k regex:Li2ELi8ELi4ELi2ELi1ELi0ELi0Ed --launch-skip 20 -c 1 -o gpurun_out/cga_c3 python tools/prof_driver.py sim 1 > gpurun_out/ncu_a.log 2>&1; echo a=$?
HF_DRIVER=1 timeout 300 $NCU -k regex:k_cg_b --launch-skip 20 -c 1 -o gpurun_out/cgb_c3 python tools/prof_driver.py sim 1 > gpurun_out/ncu_b.log 2>&1; echo b=$?
