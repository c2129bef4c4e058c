"""One KV-head shard engine (B=2, H=1, hq=4, d=128, k=64) stepped a few times:
the configuration of tests/test_gpu_exchange.py[4], run under compute-sanitizer."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_gpu_exchange import _case, _shard_engine
case = _case(steps=3)
e, _ = _shard_engine(case, 4, 1)
e.run()
print("ok", e.metrics()["misses"])
