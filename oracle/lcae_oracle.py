"""fp64 CPU oracle for one training step of a locally-connected RICA autoencoder layer.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  The product path
(paper_1502_03409_b200/ and its CUDA library) never imports, links or calls it,
and this module imports nothing from the product package.

What it computes (§3.1 eq. "RICA"):

    min_{W,alpha,b}  sum_i || W^T (alpha W x^(i)) + b - x^(i) ||_2^2  +  lambda sqrt((alpha W x^(i))^2)
    subject to ||W^(k)||_2 = 1 for every filter row k

applied independently to every receptive field of an untied (locally
connected) layer ("untied convolutional layers"; PAPER.md:118
"allowing receptive fields to be trained independently"), with the readings
of SURVEY.md §0 / DESIGN.md "Readings":

  R1  J = sum_f sum_i [ ||W_f^T h + b_f - x||^2 + lambda sum_G sqrt(eps + sum_{j in G} h_j^2) ],
      h = alpha_f W_f x (eps smoothing: SPEC.md:94, :138).
  R2  pool group g (consecutive filters); g = 1 is exactly the paper's lambda sqrt((alpha W x)^2).
  R3  the decoder uses h (pre-pool); the pooled code p = s_G is the layer's output.
  R4  alpha: one scalar per field, clamped >= alpha_min; b: per-field n-vector, reconstruction only.
  R5  SGD (optional momentum) then row projection.
  R6  sums over batch and fields, no 1/m (PAPER.md:88 sum_i).
  R7  grid = (H - rf)/stride + 1, exact; fields row-major; patch
      flatten order (ry, rx, c) over NHWC.
  R11 dX = dJ/dx, the total derivative, overlap-added over every field covering a pixel.

Every routine is the plain definition written out, one field at a time, in
float64.  numpy matmul is the only library primitive used.

Pins (tests/test_oracle_*.py, all `-m "not gpu"`): SPEC.md:97 worked example
(tests/golden/), hand-derived gradients for that instance, SPEC.md:108 db
example, central finite differences on every coordinate,
a dense masked-matrix brute-force formulation of the whole layer, closed forms
(zero W, selection W), invariants (sign flips, in-group permutations, field
independence, batch equivariance, 1x1 grid == dense RICA), geometry and
parameter-count examples, projection examples
(SPEC.md:117-119).  No function here is "parity unpinned".
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1


class GeometryError(ValueError):
    """Non-divisible field geometry (SPEC.md:189 'geometry error stating the residue')."""


class DegenerateRowError(ArithmeticError):
    """Row norm below 1e-30 (SPEC.md:117 'degenerate-row error carrying the row index')."""


# --------------------------------------------------------------------------------------
# geometry  (SPEC.md:185-193 compute_field_grid; PAPER.md:95 footnote "72x72 grid")
# --------------------------------------------------------------------------------------
def field_grid(img_h, img_w, rf_h, rf_w, stride):
    """grid_rows = (H - fh)/stride + 1 exactly; same for cols."""
    if rf_h > img_h or rf_w > img_w:
        raise GeometryError(f"receptive field {rf_h}x{rf_w} larger than image {img_h}x{img_w}")
    if stride <= 0:
        raise GeometryError("stride must be positive")
    ry, rx = (img_h - rf_h) % stride, (img_w - rf_w) % stride
    if ry or rx:
        raise GeometryError(f"non-divisible extent: residue rows={ry} cols={rx} for stride {stride}")
    return (img_h - rf_h) // stride + 1, (img_w - rf_w) // stride + 1


def param_count(fields, k, n):
    """Per field k*n (W) + n (b) + 1 (alpha), summed."""
    return fields * (k * n + n + 1)


def field_patch(X, r, c, rf_h, rf_w, stride):
    """x_f for every sample: X[:, r*s:r*s+rf_h, c*s:c*s+rf_w, :] flattened in (ry, rx, c) order
    (SPEC.md:198 'slice its input window, flatten').  Returns float64 (m, n)."""
    m = X.shape[0]
    win = X[:, r * stride:r * stride + rf_h, c * stride:c * stride + rf_w, :]
    return np.asarray(win, dtype=np.float64).reshape(m, -1)


# --------------------------------------------------------------------------------------
# one field: objective and gradients  (PAPER.md:88 eq. RICA)
# --------------------------------------------------------------------------------------
def rica_field(W_f, alpha_f, b_f, x_f, lam, eps, g):
    """Objective terms and all gradients of one field for a batch.

    W_f (k, n), alpha_f scalar, b_f (n,), x_f (m, n) (rows are samples x^(i)).
    Returns dict with J_rec, J_sparse, p (m, k/g), h (m, k), dW (k, n),
    dalpha, db (n,), dx (m, n).  Notation follows PAPER.md:88.
    """
    W = np.asarray(W_f, dtype=np.float64)
    a = float(alpha_f)
    b = np.asarray(b_f, dtype=np.float64)
    x = np.asarray(x_f, dtype=np.float64)
    k, n = W.shape
    m = x.shape[0]
    if k % g:
        raise GeometryError(f"pool group {g} does not divide filters {k}")
    # encode: h = alpha W x                                     ("alpha W x^(i)")
    U = x @ W.T                                                  # (m, k) = W x per sample
    h = a * U
    # L2 pooling over groups of g consecutive filters + sparsity (R1/R2)
    hg = h.reshape(m, k // g, g)
    s = np.sqrt(eps + (hg * hg).sum(axis=2))                     # (m, k/g)
    J_sparse = lam * s.sum()
    # decode with offset b and residual                         ("W^T(alpha W x)+b-x"; :93 offset b)
    r = h @ W + b                                                # (m, n)
    e = r - x
    J_rec = (e * e).sum()
    # backward
    delta = 2.0 * e                                              # dJ/dr
    s_rep = np.repeat(s, g, axis=1)                              # s_{G(j)} for each filter j
    # d s_G / d h_j = h_j / s_G; at s_G = 0 (only reachable with eps = 0) the subgradient 0 is taken
    ratio = np.divide(h, s_rep, out=np.zeros_like(h), where=s_rep > 0)
    dh = delta @ W.T + lam * ratio                               # dJ/dh  (m, k)
    dW = h.T @ delta + a * (dh.T @ x)                            # decoder path + encoder path
    dalpha = float((dh * U).sum())                               # h = alpha U
    db = delta.sum(axis=0)                                       # SPEC.md:104 db = sum_i 2(recon_i - x_i)
    dx = a * (dh @ W) - delta                                    # R11 total derivative
    # dalpha_abs = sum |dh (.) U|: the scale of the rounding error of the sum dalpha (R22)
    return dict(J_rec=float(J_rec), J_sparse=float(J_sparse), p=s, h=h, U=U,
                dW=dW, dalpha=dalpha, db=db, dx=dx, dalpha_abs=float(np.abs(dh * U).sum()))


def rica_objective(W_f, alpha_f, b_f, x_f, lam, eps, g=1):
    """Scalar objective of one field; used by finite differences."""
    W = np.asarray(W_f, dtype=np.float64)
    x = np.asarray(x_f, dtype=np.float64)
    h = float(alpha_f) * (x @ W.T)
    m, k = h.shape
    s = np.sqrt(eps + (h.reshape(m, k // g, g) ** 2).sum(axis=2))
    e = h @ W + np.asarray(b_f, dtype=np.float64) - x
    return float((e * e).sum() + lam * s.sum())


# --------------------------------------------------------------------------------------
# whole layer  (SPEC.md:195-213 untied_forward / untied_train_step)
# --------------------------------------------------------------------------------------
def layer_gradients(W, alpha, b, X, geo, fields=None):
    """Loss and gradients of a whole untied layer, fields in row-major order.

    W [F][k][n], alpha [F], b [F][n], X [m][H][W][C] (NHWC).  geo: mapping with
    img_h,img_w,img_c,rf_h,rf_w,stride,pool_group,lam,eps.  `fields` (optional)
    restricts the work to the listed global field indices (W/alpha/b then hold
    exactly those fields in that order); dX then only contains their
    contributions.  Returns dict: J, J_rec, J_sparse, p [m][gr][gc][k/g] (NaN
    for fields not computed), dW, dalpha, db (per listed field), dX [m][H][W][C].
    """
    gr, gc = field_grid(geo["img_h"], geo["img_w"], geo["rf_h"], geo["rf_w"], geo["stride"])
    fl = list(range(gr * gc)) if fields is None else list(fields)
    W = np.asarray(W)
    k = W.shape[1]
    g = geo["pool_group"]
    m = X.shape[0]
    s_ = geo["stride"]
    rf_h, rf_w = geo["rf_h"], geo["rf_w"]
    dX = np.zeros(X.shape, dtype=np.float64)
    p = np.full((m, gr, gc, k // g), np.nan)
    dW = np.zeros(W.shape, dtype=np.float64)
    dalpha = np.zeros((len(fl),), dtype=np.float64)
    db = np.zeros((len(fl), W.shape[2]), dtype=np.float64)
    J_rec = 0.0
    J_sparse = 0.0
    for i, f in enumerate(fl):
        r, c = divmod(f, gc)
        x_f = field_patch(X, r, c, rf_h, rf_w, s_)
        o = rica_field(W[i], alpha[i], b[i], x_f, geo["lam"], geo["eps"], g)
        J_rec += o["J_rec"]
        J_sparse += o["J_sparse"]
        p[:, r, c, :] = o["p"]
        dW[i] = o["dW"]
        dalpha[i] = o["dalpha"]
        db[i] = o["db"]
        # overlap-add of the patch gradient into image space (R11)
        dX[:, r * s_:r * s_ + rf_h, c * s_:c * s_ + rf_w, :] += o["dx"].reshape(m, rf_h, rf_w, -1)
    return dict(J=J_rec + J_sparse, J_rec=J_rec, J_sparse=J_sparse, p=p,
                dW=dW, dalpha=dalpha, db=db, dX=dX)


def layer_forward(W, alpha, b, X, geo, fields=None):
    """Pooled code p = s_G [m][gr][gc][k/g] and loss J (LCN excluded)."""
    o = layer_gradients(W, alpha, b, X, geo, fields)
    return o["p"], o["J"]


# --------------------------------------------------------------------------------------
# update  (SPEC.md:111-129 project_row_norms / sgd_step; PAPER.md:89 unit-norm constraint)
# --------------------------------------------------------------------------------------
def project_row_norms(W):
    """Each row divided by its Euclidean norm; norm < 1e-30 -> DegenerateRowError(row)."""
    W = np.asarray(W, dtype=np.float64)
    nrm = np.sqrt((W * W).sum(axis=-1, keepdims=True))
    bad = np.argwhere(nrm[..., 0] < 1e-30)
    if bad.size:
        raise DegenerateRowError(tuple(int(v) for v in bad[0]))
    return W / nrm


def splitmix64(z):
    """SplitMix64 finaliser on Python ints (counter-based generator)."""
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def reinit_row(seed, step, field, row, n):
    """Deterministic replacement for a degenerate row (SPEC.md:125 're-randomize that row from the
    seeded RNG and renormalize'): v_t = u(seed, step, field, row, t) - 1/2, u uniform on 24 bits."""
    key = splitmix64((seed ^ (step << 40) ^ (field << 20) ^ row) & MASK64)
    v = np.array([(splitmix64((key + t) & MASK64) >> 40) / float(1 << 24) - 0.5 for t in range(n)])
    return v / np.sqrt((v * v).sum())


def sgd_update(W, alpha, b, grads, lr, momentum=0.0, velocity=None, alpha_min=1e-8,
               seed=0, step=0, field_ids=None):
    """velocity <- mu v - lr grad; theta += velocity; W rows projected to unit norm; alpha clamped
    (SPEC.md:121-129).  Degenerate rows are re-initialised (reinit_row).  Returns
    (W', alpha', b', velocity', n_reinit)."""
    W = np.asarray(W, dtype=np.float64)
    alpha = np.asarray(alpha, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if velocity is None:
        velocity = (np.zeros_like(W), np.zeros_like(alpha), np.zeros_like(b))
    vW = momentum * velocity[0] - lr * grads["dW"]
    va = momentum * velocity[1] - lr * grads["dalpha"]
    vb = momentum * velocity[2] - lr * grads["db"]
    Wn = W + vW
    an = np.maximum(alpha + va, alpha_min)
    bn = b + vb
    nrm = np.sqrt((Wn * Wn).sum(axis=-1))
    n_reinit = 0
    fids = list(range(W.shape[0])) if field_ids is None else list(field_ids)
    for fi, j in np.argwhere(nrm < 1e-30):
        Wn[fi, j] = reinit_row(seed, step, fids[fi], int(j), W.shape[2])
        nrm[fi, j] = 1.0
        n_reinit += 1
    Wn = Wn / nrm[..., None]
    return Wn, an, bn, (vW, va, vb), n_reinit


def step(W, alpha, b, X, geo, lr, momentum=0.0, velocity=None, alpha_min=1e-8,
         seed=0, step_index=0, fields=None):
    """One full training step: gradients at (W, alpha, b) then the projected SGD update."""
    o = layer_gradients(W, alpha, b, X, geo, fields)
    Wn, an, bn, vel, nre = sgd_update(W, alpha, b, o, lr, momentum, velocity, alpha_min,
                                      seed, step_index, fields)
    o.update(W_new=Wn, alpha_new=an, b_new=bn, velocity=vel, n_reinit=nre)
    return o
