"""Pins of oracle.philox: Random123 known-answer vectors, keep rate, and the
partition independence of the dropout masks (reading #6)."""
import json
import os

import numpy as np

from oracle import philox as PH

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_known_answer_vectors():
    for c in json.load(open(os.path.join(GOLD, "philox_kat.json")))["cases"]:
        out = PH.philox4x32_10([int(x, 16) for x in c["ctr"]], [int(x, 16) for x in c["key"]])
        assert [int(x) for x in out] == [int(x, 16) for x in c["out"]]


def test_keep_rate_and_scale():
    for p in (0.1, 0.5):
        m = PH.hidden_mask(seed=7, layer=3, tensor=1, n=5, s=256, h=256, p=p)
        keep = (m > 0).mean()
        # binomial: 65536 draws, 6 sigma
        assert abs(keep - (1 - p)) < 6 * np.sqrt(p * (1 - p) / m.size)
        assert np.allclose(m[m > 0], 1 / (1 - p))


def test_masks_depend_only_on_global_coordinates():
    """The mask of (sequence, position, feature) is the same whatever batch it
    is computed in; different sequences / layers / tensors / heads differ."""
    a = PH.layer_masks(11, 2, [4, 5], 16, 32, 4, 0.2, 0.3)
    b = PH.layer_masks(11, 2, [5], 16, 32, 4, 0.2, 0.3)
    np.testing.assert_array_equal(a["h1"][:, 1], b["h1"][:, 0])
    np.testing.assert_array_equal(a["attn"][1], b["attn"][0])
    assert not np.array_equal(a["h1"], a["h2"])
    assert not np.array_equal(a["attn"][0, 0], a["attn"][0, 1])
    assert not np.array_equal(PH.hidden_mask(11, 2, 1, 4, 16, 32, 0.3), PH.hidden_mask(11, 3, 1, 4, 16, 32, 0.3))
