for pdl in 0 1; do echo "== HF_PDL=$pdl"; HF_PDL=$pdl timeout 300 python tools/ids_probe.py c3 2>&1 | head -2; done
HF_PDL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "simulate or c3 or cg" 2>&1 | tail -3
