set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 900 python -m pytest tests/test_abi.py -q -k shim 2>&1 | tail -2
