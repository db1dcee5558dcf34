"""Network files (reference network.py:157-248: JSON structure + little-endian float64 .bin in
declaration order): files written by the reference's own save_network (tests/golden/net_*,
tests/golden/make_golden.py --only netfile) load bit-for-bit, a save/load round trip reproduces
the same bytes, and malformed files raise ConfigurationError (tests/test_network.py:208-262)."""

import json
import os
import shutil

import numpy as np
import pytest

import paper_2007_07336_b200 as P
from paper_2007_07336_b200.errors import ConfigurationError

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["net_dense_8x6", "net_conv_3x2x3x4"]


@pytest.mark.parametrize("name", CASES)
def test_loads_reference_written_file_bitwise(name):
    net = P.load_network(os.path.join(GOLD, name))
    a = np.load(os.path.join(GOLD, name + "_arrays.npz"))
    assert net.step_size == float(a["step"])
    assert np.array_equal(net.opening.weights, a["Wo"]) and np.array_equal(net.opening.bias, a["bo"])
    assert np.array_equal(net.readout.weights, a["Wr"]) and np.array_equal(net.readout.bias, a["br"])
    W = np.stack([b.weights for b in net.blocks])
    assert np.array_equal(W, a["W"] if "W" in a else a["Wc"])
    assert np.array_equal(np.stack([b.bias for b in net.blocks]), a["b"])
    assert {b.activation for b in net.blocks} == {str(a["activation"])}


@pytest.mark.parametrize("name", CASES)
def test_round_trip_reproduces_the_bytes(name, tmp_path):
    net = P.load_network(os.path.join(GOLD, name))
    P.save_network(net, str(tmp_path / name))
    with open(os.path.join(GOLD, name + ".bin"), "rb") as fh, open(tmp_path / (name + ".bin"), "rb") as gh:
        assert fh.read() == gh.read()
    with open(os.path.join(GOLD, name + ".json")) as fh, open(tmp_path / (name + ".json")) as gh:
        assert json.load(fh) == json.load(gh)


def test_malformed_files_raise(tmp_path):
    base = str(tmp_path / "n")
    for ext in (".json", ".bin"):
        shutil.copy(os.path.join(GOLD, "net_dense_8x6" + ext), base + ext)
    with open(base + ".bin", "r+b") as fh:  # truncated payload
        fh.truncate(os.path.getsize(base + ".bin") - 8)
    with pytest.raises(ConfigurationError):
        P.load_network(base)
    with open(base + ".json") as fh:
        meta = json.load(fh)
    meta["format"] = "something-else"
    with open(base + ".json", "w") as fh:
        json.dump(meta, fh)
    with pytest.raises(ConfigurationError):
        P.load_network(base)
