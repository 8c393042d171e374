timeout 1200 python -m pytest tests/test_gpu_multipass.py -x -q -k czt_fourstep_fused 2>&1 | tail -5
