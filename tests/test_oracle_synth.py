"""CPU checks of the oracle's synthetic generator (bf16 exactness, streams)."""

import numpy as np

from oracle import mlp, synth


def test_uniform_is_bf16_exact_and_bounded():
    v = synth.uniform_bf16(123, 0, 4096, 0.5)
    assert np.array_equal(v, synth.to_bf16(v))
    assert np.all(np.abs(v) <= 0.5)
    assert abs(float(v.mean())) < 0.02


def test_counter_based_slices_agree():
    whole = synth.uniform_bf16(7, 0, 1000, 1.0)
    part = synth.uniform_bf16(7, 400, 100, 1.0)
    assert np.array_equal(whole[400:500], part)


def test_expert_streams_independent():
    a, _ = synth.expert_weights(1, 0, 256, 512)
    b, _ = synth.expert_weights(1, 1, 256, 512)
    assert not np.array_equal(a, b)
    assert abs(np.corrcoef(a.ravel(), b.ravel())[0, 1]) < 0.02


def test_expert_forward_shapes_and_scale():
    w1, w2 = synth.expert_weights(3, 2, 256, 1024)
    x = synth.request_inputs(9, 0, 64, 256)
    y = mlp.expert_forward(x, w1, w2)
    assert y.shape == (64, 256)
    assert 0.05 < float(np.std(y)) < 5.0
