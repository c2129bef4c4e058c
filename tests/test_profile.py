"""Head profiling (§8f rank 4): clo_profile_heads against the compiled
reference's profile_heads (profiler.cpp:19-125) on traces recorded by the
reference's own generator. CPU: the similarity profile and the provided-
importance path (no GPU work) are bit-exact. GPU: the blend fit's importance
(full / streaming / exact top-k attention in float64 on the device) agrees to
1e-9 and yields the same partition plan."""
import numpy as np
import pytest

from oracle.bind import Reference
from paper_2511_14510_b200 import _lib
from paper_2511_14510_b200.profile import plan_partition, profile_heads

needs_ref = pytest.mark.skipif(not Reference.available(), reason="reference library not built")


def _probes(tmp_path, n=2, L=3, hq=8, hkv=2, d=32, n_prompt=200, steps=6):
    paths = []
    for i in range(n):
        p = tmp_path / f"probe{i}.bin"
        Reference().record_synthetic_trace(p, L, hq, hkv, d, n_prompt, steps, d_model=48, sigma_step=0.05,
                                           seed=21 + i, width=8)
        paths.append(p)
    return paths


@needs_ref
def test_provided_importance_profile_is_bit_exact(tmp_path):
    paths = _probes(tmp_path)
    rng = np.random.default_rng(4)
    prov = rng.uniform(0, 1, (3, 2, 4))
    want = Reference().profile_heads(paths, provided=prov, eta=0.7, p=2.0, epsilon=0.05)
    got = profile_heads(paths, provided_importance=prov, eta=0.7, p=2.0, epsilon=0.05)
    for l in range(3):
        for g in range(2):
            e = got[l][g]
            np.testing.assert_array_equal(e.q_importance, want["q_importance"][l, g])
            assert e.kv_importance == want["kv_importance"][l, g]
            assert e.s_hat == want["s_hat"][l, g]
            assert e.tau == want["tau"][l, g]
            assert e.difficulty == want["difficulty"][l, g]


def test_profile_errors(tmp_path):
    with pytest.raises(_lib.ArgumentError):
        profile_heads([])
    if Reference.available():
        paths = _probes(tmp_path, n=1)
        with pytest.raises(_lib.ConfigError):
            profile_heads(paths, provided_importance=np.full((3, 2, 4), 1.5))
        with pytest.raises(_lib.ConfigError):
            profile_heads(paths, provided_importance=np.zeros((2, 2, 4)))


@pytest.mark.gpu
@needs_ref
def test_blend_fit_profile_matches_reference(tmp_path):
    paths = _probes(tmp_path)
    kw = dict(blend_sequences=2, blend_steps=4, topk=16, sink=4, recent=16)
    want = Reference().profile_heads(paths, **kw)
    got = profile_heads(paths, blend_sequences=2, blend_steps=4, topk=16, sink_tokens=4, recent_tokens=16)
    imp = np.array([[e.q_importance for e in layer] for layer in got])
    np.testing.assert_allclose(imp, want["q_importance"], rtol=0, atol=1e-9)
    assert (imp > 0).any() and (imp < 1).any()  # the fit is not degenerate
    s_hat = np.array([[e.s_hat for e in layer] for layer in got])
    np.testing.assert_array_equal(s_hat, want["s_hat"])
    for key in ("tau", "difficulty"):
        np.testing.assert_allclose(np.array([[getattr(e, key) for e in layer] for layer in got]), want[key],
                                   rtol=0, atol=1e-9)
    plan, n_p, _ = plan_partition(got, t_comp_s=5e-5, pcie_bw=2e10, mem_head_bytes=2 * 16 * 32 * 2)
    want_pers, want_np, _ = Reference().plan_partition(np.ascontiguousarray(want["difficulty"]), 5e-5, 2e10,
                                                       2 * 16 * 32 * 2)
    assert n_p == want_np
    assert plan.layers == [[g for g in range(2) if want_pers[l, g]] for l in range(3)]
