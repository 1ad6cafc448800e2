set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/mb_resident.cu && timeout 120 /tmp/mb > gpurun_out/mb_resident.txt 2>&1; echo mb=$?
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
HF_DRIVER=1 timeout 600 $NCU -k regex:Li8ELi3ELi2ELi1E --launch-skip 10 -c 1 -o gpurun_out/cga_512 python tools/prof_driver.py sim512 1 > gpurun_out/ncu_a512.log 2>&1; echo a512=$?
for tool in racecheck synccheck; do
  HF_DRIVER=1 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest -x -q -m gpu \
    "tests/test_gpu_parity.py::test_apply_matches_assembled" "tests/test_gpu_parity.py::test_simulate_c1" "tests/test_gpu_parity.py::test_cg_matches_oracle" \
    > gpurun_out/sanitizer_$tool.log 2>&1; echo $tool=$?
done
