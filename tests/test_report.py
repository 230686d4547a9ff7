"""Cost model (cost_model.hpp) against the reference's acceptance criteria 1, 2
and 7 (acceptance.cpp:61-131, :460-512), and the run report (pipeline.hpp) on
the device."""
import numpy as np
import pytest

from paper_2604_16864_b200 import report as R


def cp(sk, sv, L=4096, D=128, B=64):
    return R.CostParams(L, D, B, sk, sv)


def test_cost_constants_acceptance_criterion_1():
    assert abs(R.compression_ratio(cp(.75, .75), False) - 1.49) < 0.005
    assert abs(R.compression_ratio(cp(1, 1), False) - 1.78) < 0.005
    assert R.prefill_speedup(cp(.75, .75)) == 1.6
    assert R.prefill_speedup(cp(1, 1)) == 2.0
    assert R.decode_speedup(cp(.5, .5)) == 32.0 / 25.0
    assert abs(R.decode_speedup(cp(1, 1)) - 1.78) < 0.005
    assert R.compression_ratio(cp(.25, .25), True) == 1.0 / 0.8907470703125
    t = R.design_space_table()
    assert [r["config"] for r in t] == ["Naive", "Trans-K", "Trans-V", "Trans-Both"]
    assert [r["sparse_operands"] for r in t] == [["Q", "P"], ["K", "P"], ["Q", "V"], ["K", "V"]]
    assert [r["ideal_decode"] for r in t] == [1.0, 1.5, 1.5, 2.0] and all(r["ideal_prefill"] == 2.0 for r in t)


@pytest.mark.parametrize("sk", [0.0, 0.25, 0.5, 0.75, 1.0])
@pytest.mark.parametrize("sv", [0.0, 0.25, 0.5, 0.75, 1.0])
def test_measured_ratio_equals_exact_model_criterion_2(sk, sv):
    """measure_size of the pool geometry (host-computable, pruner.hpp:106-108)
    over the quarter grid at L=4096, D=128, B=64: rel err < 1e-12."""
    L, D, B = 4096, 128, 64
    nb = L // B

    def size(s):
        sparse = int(np.floor(s * nb))
        dense = nb - sparse
        return 2 * nb + dense * B * D * 2 + sparse * (B * D // 2) * 2 + sparse * (B * D // 16) * 2
    measured = 2.0 * L * D * 2.0 / (size(sk) + size(sv))
    model = R.compression_ratio(cp(sk, sv), True)
    assert abs(measured - model) / model < 1e-12


def test_analytic_flops_identity_criterion_7():
    """flops = n_q * L * D * (4 - S_K - S_V) for a non-causal full-length workload
    (acceptance.cpp:460-512) from the host closed form of flop_and_byte_count."""
    from paper_2604_16864_b200.hierasparse import flop_count
    L, D, B = 1024, 128, 64
    nb = L // B
    for sk, sv in [(0, 0), (.5, 1), (1, 1), (.25, .75)]:
        kd = [1] * (nb - int(sk * nb)) + [0] * int(sk * nb)
        vd = [1] * (nb - int(sv * nb)) + [0] * int(sv * nb)
        f = flop_count(kd, vd, B, D, L, 0, causal=False)
        assert f == round(L * L * D * (4 - sk - sv))
        assert f * R.prefill_speedup(cp(sk, sv, L, D, B)) == 4 * L * L * D


def test_config_errors():
    from paper_2604_16864_b200 import ConfigError
    with pytest.raises(ConfigError):
        R.compression_ratio(cp(1.5, 0), True)
    with pytest.raises(ConfigError):
        R.RunConfig(seq_len=100).validate()
    assert R.main(["cost", "--s-key", "2"]) == 2


@pytest.mark.gpu
def test_run_pipeline_report():
    rep = R.run_pipeline(R.RunConfig(seq_len=2048, heads=2, gqa_group=4, s_key_prefill=.5, s_value_prefill=1.0,
                                     s_key_decode=1.0, s_value_decode=1.0))
    assert abs(rep["compression"]["r_comp_measured"] - rep["compression"]["r_comp_model_exact"]) < 1e-9
    assert rep["accuracy"]["prefill_vs_decompressed"]["max_abs"] < 2e-2
    assert rep["accuracy"]["decode_vs_decompressed"]["max_abs"] < 2e-2
    assert rep["b200"]["prefill_ms"] > 0 and rep["b200"]["decode_ms"] > 0
