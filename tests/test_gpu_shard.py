"""KV-head sharding on the CUDA engine: engines serving disjoint KV-head
blocks (EngineConfig.kv_head_offset keeps the global per-head sign-hash seeds)
reproduce the unsharded engine's selections exactly and its outputs for
their heads to float rounding — the per-rank work of configs[3]; the all-gather itself is covered
on CPU by tests/test_multiprocess.py."""
import dataclasses

import numpy as np
import pytest

from paper_2511_14510_b200 import DecodeEngine, PartitionPlan, profiles_from_arrays
from paper_2511_14510_b200.dist import kv_head_shard
from paper_2511_14510_b200.workload import HeadSlice
from tests.engine_harness import make_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4])
def test_kv_head_shards_match_unsharded_engine(world):
    case = make_case(L=3, hq=16, hkv=4, d=128, n_prompt=600, steps=6, k=64, batch=2, kv_dtype="bf16",
                     sink=4, recent=64)
    cfg, wl = case["cfg"], case["wl"]
    full = DecodeEngine(cfg, profiles_from_arrays(case["tau"], case["qimp"]), case["plan"], wl)
    full.run()
    want = np.stack(full.collected_outputs())  # [steps][B][L][hq][d]
    s = cfg.shape
    for rank in range(world):
        sh = kv_head_shard(s.num_q_heads, s.num_kv_heads, world, rank)
        sl = slice(sh.kv0, sh.kv0 + sh.n_kv)
        scfg = dataclasses.replace(cfg, shape=dataclasses.replace(s, num_q_heads=sh.n_q, num_kv_heads=sh.n_kv),
                                   kv_head_offset=sh.kv0)
        plan = PartitionPlan(layers=[[g - sh.kv0 for g in heads if sh.kv0 <= g < sh.kv0 + sh.n_kv]
                                     for heads in case["plan"].layers])
        eng = DecodeEngine(scfg, profiles_from_arrays(case["tau"][:, sl], case["qimp"][:, sl]), plan,
                           HeadSlice(wl, sh.kv0, sh.n_kv, sh.q0, sh.n_q))
        eng.run()
        got = np.stack(eng.collected_outputs())
        # float rounding only: the attention kernel's warp split depends on the
        # shard's head count (selections below are bit-exact)
        np.testing.assert_allclose(got, want[:, :, :, sh.q0:sh.q0 + sh.n_q], rtol=1e-5, atol=1e-6)
        for l in range(s.num_layers):
            for g in range(sh.n_kv):
                a, b = eng.head(l, g), full.head(l, sh.kv0 + g)
                assert a["hits"] == b["hits"] and a["misses"] == b["misses"]
                np.testing.assert_array_equal(a["entry_indices"], b["entry_indices"])
