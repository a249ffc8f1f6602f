"""The shared input generator: numpy and torch produce identical values; values are bf16-exact."""
import numpy as np
import torch

import synth


def test_counter_numpy_equals_torch():
    for stream in (synth.S_WQKV, synth.S_KHIST):
        for off in (0, (1 << 33) + 17):
            a = synth.counter_values(4791, stream, (37, 53), off, scale_pow2=3)
            b = synth.counter_values_torch(4791, stream, (37, 53), off, scale_pow2=3).numpy()
            np.testing.assert_array_equal(a, b)


def test_values_exact_in_bf16_and_moments():
    a = synth.counter_values(1, synth.S_XPRE, (200000,))
    np.testing.assert_array_equal(synth.round_to_bf16(a), a)
    t = torch.from_numpy(a).to(torch.bfloat16).float().numpy()
    np.testing.assert_array_equal(t, a)
    assert abs(a.mean()) < 0.01 and 0.95 < a.var() < 1.03
    k = np.round(a * 64).astype(int)
    assert k.min() == -110 and k.max() == 110


def test_page_tables_distinct_and_cover():
    t, used = synth.page_tables(3, [17, 32, 1, 0, 100], 16, 20)
    flat = t[t >= 0]
    assert len(set(flat.tolist())) == len(flat) == used == 2 + 2 + 1 + 0 + 7
    assert flat.max() < 20
