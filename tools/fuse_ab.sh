for f in 0 1; do echo "== HF_FUSE_AB=$f"; HF_FUSE_AB=$f timeout 300 python tools/ids_probe.py c3 2>&1 | head -2; done
timeout 600 python -m pytest tests/test_gpu_fused.py -x -q 2>&1 | tail -5
