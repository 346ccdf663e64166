"""Golden values from the paper / SPEC worked examples (tests/golden/paper_pins.json)."""
import json
import math
import os

import oracle

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))


def test_param_count_golden():
    d = G["params_3d_point_net"]["arch"]
    assert oracle.num_params(oracle.make_arch(d[0], d[1], len(d) - 2)) == G["params_3d_point_net"]["value"]


def test_bce_golden():
    for (z, y, a, b), v in zip(G["bce_kats"]["cases"], G["bce_kats"]["values"]):
        assert abs(oracle.weighted_bce(z, y, a, b) - v) < 1e-6


def test_sigmoid_golden():
    assert abs(1 / (1 + math.exp(-3)) - G["sigmoid_3"]["value"]) < 1e-6
