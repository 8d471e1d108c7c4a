"""Parity metrics of SURVEY 8(c) "Parity definitions".

Radiance: per channel max_i |q_gpu - q_ref| / max_i |q_ref|          <= 1e-2
Gradients: per matrix max |G_gpu - G_ref| / max |G_ref|              <= 3e-2
Post-Adam: per matrix, over entries whose gradients agree in sign (and,
           within 100 eps_A of zero, within half their magnitude; R26),
           max |w_gpu - w_ref| / max |w_ref|                         <= 3e-2
           (other entries: <= 1% and each |G_ref| <= 3e-2 max|G_ref|)
The tolerances are north_star's (BASELINE.json)."""
import numpy as np

OFF = [0, 4096, 8192, 12288, 16384, 20480, 20672]
TOL_RADIANCE = 1e-2
TOL_GRAD = 3e-2
TOL_PARAM = 3e-2


def offsets_w(hw):
    """Matrix offsets of the logical layout at hidden width hw (W0 hw x 64,
    W1..W4 hw x hw, W5 3 x hw)."""
    sizes = [hw * 64] + [hw * hw] * 4 + [3 * hw]
    return [int(x) for x in np.concatenate([[0], np.cumsum(sizes)])]


def offsets_d(hw, nh):
    """Matrix offsets at hidden width hw with nh hidden layers (depth variants):
    W0 hw x 64, W1..W_{nh-1} hw x hw, W_nh 3 x hw."""
    sizes = [hw * 64] + [hw * hw] * (nh - 1) + [3 * hw]
    return [int(x) for x in np.concatenate([[0], np.cumsum(sizes)])]


def per_matrix_err_d(a, b, off):
    """per_matrix_err over an arbitrary number of matrices (offsets `off`)."""
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return [float(np.max(np.abs(a[off[i]:off[i + 1]] - b[off[i]:off[i + 1]])) /
                  max(np.max(np.abs(b[off[i]:off[i + 1]])), 1e-30)) for i in range(len(off) - 1)]


def radiance_err(q_gpu, q_ref):
    q_gpu = np.asarray(q_gpu, np.float64); q_ref = np.asarray(q_ref, np.float64)
    return [float(np.max(np.abs(q_gpu[:, c] - q_ref[:, c])) / max(np.max(np.abs(q_ref[:, c])), 1e-30))
            for c in range(3)]


def per_matrix_err(a, b, off=OFF):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    OFF = off
    out = []
    for i in range(6):
        x, y = a[OFF[i]:OFF[i + 1]], b[OFF[i]:OFF[i + 1]]
        out.append(float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-30)))
    return out


ADAM_EPS = 1e-8  # reading R11


def post_adam_err(w_gpu, w_ref, g_gpu, g_ref, off=OFF):
    """Per-matrix post-Adam error over agreeing entries, plus the statistics of
    the others (fraction, and worst |G_ref| / max|G_ref| among them).

    g_gpu / g_ref are batch-MEAN gradients.  Adam's first step is sign-like,
    dw = -lr g / (|g| + eps_A): where both |g| exceed 100 eps_A the two steps
    differ by < 0.01 lr whenever the signs agree, but where one side is within
    100 eps_A of zero the step is a steep function of g.  So an entry counts
    with the sign flips (reading R26) if the signs differ, or if one side is
    within 100 eps_A of zero and the two gradients differ by more than half
    of the oracle's (a near-cancellation, possible only where |g_ref| is
    within the gradient tolerance of zero); those keep SURVEY 8(c)'s bounds
    (<= 1% of the entries, each |G_ref| <= 3e-2 max|G_ref|).  Entries with an
    exactly zero gradient on both sides (inactive one-blob bins, dead ReLUs)
    agree."""
    w_gpu = np.asarray(w_gpu, np.float64); w_ref = np.asarray(w_ref, np.float64)
    g_gpu = np.asarray(g_gpu, np.float64); g_ref = np.asarray(g_ref, np.float64)
    OFF = off
    errs, flips, worst = [], 0, 0.0
    for i in range(len(OFF) - 1):
        s = slice(OFF[i], OFF[i + 1])
        a, b = g_gpu[s], g_ref[s]
        near = np.minimum(np.abs(a), np.abs(b)) <= 100 * ADAM_EPS
        flip = (np.sign(a) != np.sign(b)) | (near & (np.abs(a - b) > 0.5 * np.abs(b)))
        agree = ~flip
        gmax = max(np.max(np.abs(b)), 1e-30)
        flips += int(flip.sum())
        if flip.any():
            worst = max(worst, float(np.max(np.abs(b[flip])) / gmax))
        d = np.abs(w_gpu[s] - w_ref[s])[agree]
        errs.append(float(d.max() / max(np.max(np.abs(w_ref[s])), 1e-30)) if d.size else 0.0)
    return errs, flips / float(len(w_ref)), worst


def fp16_ulp(x):
    """ulp of the fp16 number nearest to x (subnormal spacing 2^-24)."""
    x = np.abs(np.asarray(x, np.float64))
    e = np.floor(np.log2(np.maximum(x, 2.0 ** -14)))
    return 2.0 ** (e - 10)


def assert_support_sets(got, ref):
    """One-blob support sets of the encodings (columns 36..55) agree in both
    directions: every bin the oracle puts clearly inside the kernel's support
    (value > 2^-12) is active on the GPU, and every bin active on the GPU is
    inside the oracle's support (value > 0).  Between the two thresholds lie
    the |x| = 1 ties, where the quartic is ~0 and the fp16 value may round
    either way (reading R17)."""
    got = np.asarray(got, np.float64)[:, 36:56]
    ref = np.asarray(ref, np.float64)[:, 36:56]
    act_gpu = got > 0
    miss = (ref > 2.0 ** -12) & ~act_gpu
    extra = act_gpu & ~(ref > 0)
    assert not miss.any(), f"{int(miss.sum())} oracle-active bins inactive on the GPU, first at {np.argwhere(miss)[:3]}"
    assert not extra.any(), f"{int(extra.sum())} GPU-active bins outside the oracle support, first at {np.argwhere(extra)[:3]}"
