"""Test helper (reading C-A32): the error the oracle predicts for a sharded run's quantised mode swaps.
Used by the loopback (one GPU) and the NCCL (several GPUs) sharded-stem tests."""
import numpy as np

from oracle import contract
from oracle.plan import load


def predicted_swap_error(plan, rep, ref, preset):
    """Reading C-A32: the codec error of each quantised swap, propagated to the result by the
    oracle.  For swap i the oracle's stem tensor entering step i is laid out as the sender sees it
    (rank bits = shard_before, then send_layout), quantised and dequantised by the ORACLE codec
    (Eq. 1, groups of g reals along the innermost modes, preset `preset`), and the error e_i is
    pushed through the rest of the network (contract(..., override) — the contraction is linear
    in every node, so the root receives L_i(e_i)).  Independent swap errors add in quadrature:
    pred^2 = sum_i |L_i(e_i)|^2 / |ref|^2."""
    from oracle import codec
    P = load(plan)
    nl = len(P.tensors)
    qmin, qmax, ex, g, rnd = codec.PRESETS[preset]
    sw = [i for i, st in enumerate(rep["steps"]) if st.get("quant")]
    if not sw:
        return 0.0
    stem_in = {}
    for i in sw:
        st = rep["steps"][i]
        u, v = P.tree[st["node"] - nl]
        stem_in[i] = v if u == st["branch"] else u
    rec = {stem_in[i]: None for i in sw}
    contract.contract(P, 0, record=rec)
    tot = 0.0
    for i in sw:
        st = rep["steps"][i]
        lab, t = rec[stem_in[i]]
        glay = list(st["shard_before"]) + list(st["send_layout"])
        x = np.transpose(t, [lab.index(l) for l in glay])
        re = np.stack([x.real, x.imag], axis=-1).astype(np.float32).reshape(-1)
        # Table 1 int8 preset: one group per destination chunk (the reals after the rank bits and the
        # swapped-in modes)
        gi = g if g is not None else 2 << (len(st["send_layout"]) - len(st["swap_out_pos"]))
        c, sc, ze = codec.quantize(re, qmin, qmax, ex, gi, rnd)
        y = codec.dequantize(c, sc, ze, ex, gi).astype(np.float64).reshape(x.shape + (2,))
        e = (y[..., 0] + 1j * y[..., 1]) - x
        e = np.transpose(e, [glay.index(l) for l in lab])
        le = contract.contract(P, 0, override={stem_in[i]: (lab, e)})
        tot += float(np.sum(np.abs(le) ** 2))
    return float(np.sqrt(tot) / np.linalg.norm(ref))
