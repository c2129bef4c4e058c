timeout 1200 python -m pytest tests/test_gpu_edge_cases.py -q 2>&1 | tail -30
