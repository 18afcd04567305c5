"""Top-K stimuli per unit — TEST INFRASTRUCTURE ONLY (see lcae_oracle.py header for who may import oracle/).

SPEC.md:500-508 top_k_stimuli(activations, K): per neuron, the K (image id, value) pairs with the largest
values, sorted by value descending, ties broken by the lower image id; K > N returns all N.
PAPER.md:158 ("we show the top 5 stimuli for some example neurons"). Written as the plain definition: a full
sort of every unit's column with that ordering, then the first K. numpy lexsort is the only primitive.
"""
import numpy as np


def top_k_stimuli(acts, K):
    """acts [N images][U units] -> (vals [U][min(K, N)] float64, ids [U][min(K, N)] int64)."""
    acts = np.asarray(acts, dtype=np.float64)
    N, U = acts.shape
    kk = min(K, N)
    ids = np.arange(N)
    vals_out = np.zeros((U, kk))
    ids_out = np.zeros((U, kk), dtype=np.int64)
    for u in range(U):
        order = np.lexsort((ids, -acts[:, u]))   # primary: value descending; secondary: id ascending
        ids_out[u] = order[:kk]
        vals_out[u] = acts[order[:kk], u]
    return vals_out, ids_out
