"""Pins of the top-K stimuli oracle (SPEC.md:500-508 examples; brute force on tiny inputs)."""
import numpy as np

from oracle import top_k_stimuli


def test_spec_example_k1():
    # K=1, single neuron, values (0.1, 0.9, 0.5) -> image 1, value 0.9
    v, i = top_k_stimuli(np.array([[0.1], [0.9], [0.5]]), 1)
    assert i.tolist() == [[1]] and v.tolist() == [[0.9]]


def test_spec_example_ties():
    # all-equal values, K=3 -> images 0, 1, 2 by the tie rule
    v, i = top_k_stimuli(np.full((7, 1), 0.25), 3)
    assert i.tolist() == [[0, 1, 2]] and v.tolist() == [[0.25, 0.25, 0.25]]


def test_k_larger_than_n_returns_all_sorted():
    v, i = top_k_stimuli(np.array([[0.3], [0.7]]), 5)
    assert i.tolist() == [[1, 0]] and v.tolist() == [[0.7, 0.3]]


def test_brute_force_small():
    # every K-subset ordering checked against an explicit enumeration on a tiny quantised matrix
    rng = np.random.default_rng(3)
    acts = rng.integers(0, 4, size=(6, 5)).astype(np.float64)
    for K in (1, 2, 4, 6):
        v, i = top_k_stimuli(acts, K)
        for u in range(acts.shape[1]):
            best = sorted(range(6), key=lambda s: (-acts[s, u], s))[:K]
            assert i[u].tolist() == best
            assert v[u].tolist() == [acts[s, u] for s in best]
            # the chosen set dominates every other image
            for s in set(range(6)) - set(best):
                assert all((acts[b, u], -b) > (acts[s, u], -s) for b in best)
