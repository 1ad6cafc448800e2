# round 2 (final state): bench line, ncu launch list of the bench command, ncu --set full of PCG
# kernels A and B (C3 and 512^3), the single-reduction PCG kernel (C3) and the 512^3 apply,
# (host-loop driver: ncu does not follow kernels inside conditional graph nodes).  Large reports are reduced to CSV on the box (gpurun copies back <= 64 MiB).
set -x
timeout 1200 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo bench=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_under_ncu.log 2>&1; echo launches=$?
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base mangled"
cap() {   # name, env, kernel regex, skip, driver args...
  name=$1; shift; envs=$1; shift; rx=$1; shift; skip=$1; shift
  env $envs timeout 600 $NCU -k regex:$rx --launch-skip $skip -c 1 -o gpurun_out/$name "$@" > gpurun_out/$name.log 2>&1; echo $name=$?
  ncu -i gpurun_out/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
  ncu -i gpurun_out/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/$name.sass.csv 2>/dev/null
  gzip -f gpurun_out/$name.sass.csv
  rm -f gpurun_out/$name.ncu-rep
}
cap r02_cga_c3 HF_DRIVER=1 Li2ELi8ELi4ELi2ELi1ELi0ELi0Ed 20 python tools/prof_driver.py sim 1
cap r02_cgb_c3 HF_DRIVER=1 k_cg_b 20 python tools/prof_driver.py sim 1
cap r02_cg1_c3 "HF_DRIVER=1 CG_VARIANT=1" Li8ELi3ELi4ELi4ELi0 20 python tools/prof_driver.py sim 1
cap r02_cga_512 HF_DRIVER=1 Li4ELi8ELi3ELi2ELi1ELi0ELi0Ed 10 python tools/prof_driver.py sim512 1
cap r02_cgb_512 HF_DRIVER=1 k_cg_b 10 python tools/prof_driver.py sim512 1
cap r02_apply512 HF_X=0 Li4ELi8ELi4ELi0ELi0ELi0ELi0Ed 1 python tools/prof_driver.py apply512 2
# compute-sanitizer: closed on the GPU pool late in round 2 (profiles/r02_sanitizer_*.log are
# from the earlier round-2 run on the same kernels)
du -sh gpurun_out; ls -la gpurun_out | tail -40
