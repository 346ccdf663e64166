"""CPU checks behind the tolerance readings of DESIGN.md (oracle only, no GPU).

R46: the scaled random test weights (gpu_helpers.SCALE) are chosen by a
property of the oracle alone: at that gain the bf16 network (ORA_BF16_EMU:
bf16 weights and activations) stays within BASELINE.json's 2e-2 sigmoid
bound of the fp64 network, so the plain P2 bound can be asserted on every
row of the kernel's output.  At gain 2.5 the 6-layer c4 net's own bf16 gap
already exceeds the bound (what R47 accounts for at trained weights)."""
import numpy as np
import pytest

import nbgen
import oracle
from gpu_helpers import SCALE, scaled_params, sigmoid


def _gap(name, scale, n):
    cfg = nbgen.CONFIGS[name]
    a = oracle.arch_of(cfg)
    q = nbgen.make_queries(cfg, nbgen.TAG_EVAL, 0, n).numpy()
    th = scaled_params(cfg, 4, scale=scale).double().numpy()
    z64 = oracle.forward(a, th, q)
    ze = oracle.forward(a, th, q, oracle.BF16_EMU)
    return np.abs(sigmoid(ze) - sigmoid(z64)).max(), z64.std()


@pytest.mark.parametrize("name,n", [("c2", 1 << 14), ("c3", 1 << 12), ("c4", 1 << 12), ("c5", 1 << 11)])
def test_scaled_gain_keeps_bf16_network_within_p2(name, n):
    gap, std = _gap(name, SCALE[name], n)
    assert gap < 1.5e-2, gap          # margin below the 2e-2 bound for the kernel's own rounding order
    assert std > 0.15                 # logits still spread (not a trivially flat network)


def test_gain_2p5_breaks_the_bf16_network_for_c4():
    gap, _ = _gap("c4", 2.5, 1 << 12)
    assert gap > 2e-2
