"""bench.py's accounting on CPU: the algorithmic attention FLOPs behind `roofline.achieved`
equal SURVEY §8(d)'s figures, and the DRAM-traffic lookup returns the committed ncu capture
for the headline kernel (profiles/attn_traffic.json)."""

import importlib.util
import os

import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_under_test", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)  # defines functions only; main() is not run
    return mod


def test_attention_flops_match_survey(bench):
    C = bench.CONFIGS
    # c1 36.24 GFLOP per 3-block rollout, c2 565.2 TFLOP per 7-block rollout
    assert bench.attn_flops_per_rollout(C["c1"]) == pytest.approx(36.24e9, rel=1e-3)
    assert bench.attn_flops_per_rollout(C["c2"]) == pytest.approx(565.2e12, rel=1e-3)
    # c3: 423.9 TFLOP for the block generated with b = 20 cached blocks
    c3 = C["c3"]
    last = bench.attn_flops_per_rollout(c3) - bench.attn_flops_per_rollout(dict(c3, blocks=20))
    assert last == pytest.approx(423.9e12, rel=1e-3)
    # c4: 448.56 GFLOP x (b + 1) per layer-pass
    c4 = dict(C["c4"], layers=1, blocks=1)
    assert bench.attn_flops_per_rollout(c4) / (len(bench.STEPS) + 1) == pytest.approx(448.56e9, rel=1e-3)


def test_traffic_lookup_is_the_committed_capture(bench):
    traffic, note = bench.attn_traffic("c2", 1)
    assert traffic is not None and 0.9 < traffic / 230031360 < 1.1  # ~= algorithmic bytes
    assert "ncu" in note
    assert bench.attn_traffic("c2", 8)[0] is not None  # the 8-rank (grouped plan) launch too
