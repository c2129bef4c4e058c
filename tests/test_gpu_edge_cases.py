"""Edge cases of the decode path, CUDA engine vs the CPU oracle (same harness
as test_gpu_engine.py: bit-exact selections/decisions/rows, outputs within
tolerance)."""
import numpy as np
import pytest

from tests.engine_harness import gpu_engine, make_case, run_and_compare

pytestmark = pytest.mark.gpu


def test_k_equals_prompt_selects_everything(oracle):
    case = make_case(n_prompt=48, k=48, steps=5, sink=2, recent=8)
    g, o, _ = run_and_compare(case, oracle)
    assert list(g.head(1, 0)["entry_indices"][:3]) == [0, 1, 2]


def test_k_one(oracle):
    run_and_compare(make_case(k=1, steps=6), oracle)


@pytest.mark.parametrize("sink,recent", [(0, 0), (0, 16), (4, 0), (8, 200)])
def test_window_shapes(oracle, sink, recent):
    run_and_compare(make_case(sink=sink, recent=recent, n_prompt=120, steps=6, k=8), oracle)


@pytest.mark.parametrize("bits", [8, 64, 128, 192, 512])
def test_hash_widths(oracle, bits):
    run_and_compare(make_case(hash_bits=bits, steps=6), oracle)


@pytest.mark.parametrize("bits", [64, 192, 320])
def test_hash_widths_odd_segment_length(oracle, bits):
    """Odd code words per row and an odd n_prompt + steps: every other
    segment's codes would start 8-byte aligned without the engine's even
    per-segment code stride (the TMA score kernel's bulk copies need 16)."""
    case = make_case(hash_bits=bits, n_prompt=97, steps=6)
    assert (97 + 6) % 2 == 1 and case["cfg"].batch * case["cfg"].shape.num_kv_heads >= 2
    run_and_compare(case, oracle)


def test_aliased_host_store_rejects_layer_dependent_rows():
    """layer_stride 0 aliases one host matrix across layers: a step whose new
    K/V rows differ between layers is a ContractError, not silent corruption."""
    from paper_2511_14510_b200._lib import ContractError
    case = make_case(L=3, steps=3, alias_layers=True)
    wl = case["wl"]
    g = gpu_engine(case)
    g.prefill()
    g.decode_step()  # identical rows across layers: fine
    g.metrics()  # synchronises; raises a deferred device error
    base = wl.step_new_kv

    def skewed(t):
        k, v = base(t)
        k = k.copy()
        k[:, 2] = k[:, 0] + 1.0  # f32 rows: layer 2 appends a different key
        return k, v
    wl.step_new_kv = skewed
    with pytest.raises(ContractError, match="aliases"):
        g.decode_step()  # synchronises: the device-side check surfaces here


@pytest.mark.parametrize("victim", [0, 3, 8, 40, -1])
@pytest.mark.parametrize("interleaved", [False, True])
def test_row_pool_sizes(oracle, victim, interleaved):
    """The HBM row pool (entry + victim rows, least recently vacated evicted
    first): entries and gathered rows stay bit-exact for every pool size, and
    the PCIe rows moved equal the pool model's count (engine_harness.PoolModel)
    — from none kept (victim 0: the plain delta gather) to more than the
    working set."""
    case = make_case(steps=24, k=8, sigma_step=0.35, victim_rows=victim, interleaved=interleaved,
                     tau=0.9, kv_dtype="bf16", d=64)
    run_and_compare(case, oracle)


def test_tie_heavy_integer_keys_exact(oracle):
    # integer-valued keys and queries: exact dot products collide massively;
    # the (score desc, index asc) order decides every selection
    case = make_case(retriever="exact", steps=8, k=12, sigma_step=0.3)
    wl = case["wl"]
    for arr in (wl.prompt_k, wl.new_k):
        arr[...] = np.round(arr * 1.5)
    for arr in (wl.true_q, wl.approx_q):
        arr[...] = np.round(arr * 3)
    run_and_compare(case, oracle)


@pytest.mark.parametrize("hq,hkv", [(4, 4), (16, 2)])
def test_group_sizes_mha_and_m8(oracle, hq, hkv):
    run_and_compare(make_case(hq=hq, hkv=hkv, steps=6, d=16), oracle)


@pytest.mark.parametrize("d,kv_dtype", [(64, "bf16"), (256, "bf16"), (128, "f32"), (64, "f32")])
def test_tma_attention_shapes(oracle, d, kv_dtype):
    case = make_case(d=d, kv_dtype=kv_dtype, n_prompt=300, k=40, steps=5, sink=4, recent=64, hq=8, hkv=2)
    _, _, worst = run_and_compare(case, oracle)
    assert worst < 1e-5


def test_acceptance_criterion_4_scale(oracle):
    # acceptance_main.cpp:142-206: L=4, 4q/2kv, d=32, n=512, 200 steps,
    # always_miss, exact retriever -> worst rel-L2 <= 1e-5 against the oracle
    case = make_case(L=4, hq=4, hkv=2, d=32, n_prompt=512, steps=200, k=52, batch=1, retriever="exact",
                     always_miss=True, kv_dtype="f32", sink=4, recent=64)
    _, _, worst = run_and_compare(case, oracle, check_rows=False)
    assert worst <= 1e-5


def test_non_finite_prompt_raises_at_prefill():
    from paper_2511_14510_b200._lib import NumericError
    case = make_case(steps=2, kv_dtype="f32")
    case["wl"].prompt_v[0, 1, 0, 5, 3] = np.inf
    g = gpu_engine(case)
    with pytest.raises(NumericError):
        g.prefill()


def test_invalid_configs_raise():
    from paper_2511_14510_b200._lib import ArgumentError, ConfigError
    for kw, exc in ((dict(k=0), ArgumentError), (dict(k=97), ArgumentError),
                    (dict(always_miss=True, always_hit=True), ConfigError)):
        case = make_case(**kw)
        with pytest.raises(exc):
            gpu_engine(case)
    case = make_case(policy="prefetch_only")
    case["cfg"].policy = "lru"  # block caches are outside the path
    with pytest.raises(ConfigError):
        gpu_engine(case)


@pytest.mark.parametrize("m", [1, 2, 3, 8])
@pytest.mark.parametrize("d", [64, 128])
def test_tensor_core_attention_group_sizes(oracle, m, d):
    """The mma.sync attention (bf16, d 64/128) for every GQA group size the
    A tile carries (rows 0..m-1 hi, 8..8+m-1 lo), against the fp64 oracle."""
    case = make_case(L=2, hq=2 * m, hkv=2, d=d, n_prompt=400, steps=4, k=48, batch=2, kv_dtype="bf16",
                     sink=4, recent=64)
    run_and_compare(case, oracle)


def test_tensor_core_attention_flat_split(oracle):
    """B*H = 320 heads > 2 x 148: the attention leaves the head-aligned layout
    for the flat split (segments straddle heads, per-warp partials merged by
    the last warp of each head)."""
    case = make_case(L=2, hq=32, hkv=8, d=64, n_prompt=260, steps=3, k=32, batch=40, kv_dtype="bf16",
                     sink=4, recent=16)
    run_and_compare(case, oracle)
