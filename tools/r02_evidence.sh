# round 2 evidence: ncu --set full of PCG kernels A and B at 512^3 (backs bench c4_steps), and
# compute-sanitizer (memcheck / racecheck / synccheck) on small-grid GPU tests
set -x
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
HF_DRIVER=1 timeout 600 $NCU -k regex:Li8ELi4ELi2ELi1E --launch-skip 10 -c 1 -o gpurun_out/cga_512 python tools/prof_driver.py sim512 1 > gpurun_out/ncu_a512.log 2>&1; echo a512=$?
HF_DRIVER=1 timeout 600 $NCU -k regex:k_cg_b --launch-skip 10 -c 1 -o gpurun_out/cgb_512 python tools/prof_driver.py sim512 1 > gpurun_out/ncu_b512.log 2>&1; echo b512=$?
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest -x -q -m gpu \
    "tests/test_gpu_parity.py::test_apply_matches_assembled" "tests/test_gpu_parity.py::test_simulate_c1" "tests/test_gpu_parity.py::test_cg_matches_oracle" "tests/test_gpu_parity.py::test_batched_systems_have_their_own_pcg" \
    > gpurun_out/sanitizer_$tool.log 2>&1; echo $tool=$?
done
ls -la gpurun_out
