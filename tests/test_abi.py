"""CPU-only checks: the C-ABI library loads and exports every symbol include/lmg.h declares, and
the host-side logic (partition, protocol, hierarchy sizing, errors) matches the reference."""

import ctypes
import os
import re

import numpy as np
import pytest

from _golden import ROOT, fas

import paper_2007_07336_b200 as P
from paper_2007_07336_b200 import _lib
from paper_2007_07336_b200.multigrid import _levels_for

HEADER = os.path.join(ROOT, "include", "lmg.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(lmg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2007_07336_b200.build import build

    build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES)
    lib = _lib.load()
    assert lib.lmg_abi_version() == 1


def test_library_errors_without_device_are_loud():
    lib = _lib.load()
    n = ctypes.c_int(0)
    assert lib.lmg_num_levels(1024, 4, 64, ctypes.byref(n)) == 0 and n.value == 3
    assert lib.lmg_num_levels(1024, 1, 0, ctypes.byref(n)) == _lib.LMG_ERR_CONFIGURATION
    assert lib.lmg_num_levels(24, 4, 1, ctypes.byref(n)) == _lib.LMG_ERR_CONFIGURATION
    with pytest.raises(P.ConfigurationError):
        _lib.check(_lib.LMG_ERR_CONFIGURATION)
    with pytest.raises(P.DimensionError):
        _lib.check(_lib.LMG_ERR_DIMENSION)
    with pytest.raises(P.ProtocolError):
        _lib.check(_lib.LMG_ERR_PROTOCOL)


@pytest.mark.parametrize("n,c,thr", [(64, 4, None), (1024, 4, 64), (32, 2, 4), (4, 4, None),
                                     (128, 8, 2), (1024, 16, 4), (256, 4, 16)])
def test_level_counts_match_reference_rule(n, c, thr):
    lev = fas.DenseLevel(np.zeros((n, 1, 1)), np.zeros((n, 1)), "tanh", 1.0)
    assert _levels_for(n, c, thr) == len(fas.build_levels(lev, c, thr))
    ctyp = ctypes.c_int(0)
    assert _lib.load().lmg_num_levels(n, c, 0 if thr is None else thr, ctypes.byref(ctyp)) == 0
    assert ctyp.value == len(fas.build_levels(lev, c, thr))


def test_hierarchy_validation_is_host_side():
    net = P.random_network(16, 3, seed=0)
    hier = P.build_hierarchy(net, 4, threshold=4)
    assert [lv.num_layers for lv in hier.levels] == [16, 4]
    assert hier.levels[1].step_size == 4 * net.step_size
    assert hier.levels[1].blocks[1] is net.blocks[4]  # aliasing, multigrid.py:83-85
    with pytest.raises(P.ConfigurationError):
        P.build_hierarchy(net, 1)
    with pytest.raises(P.ConfigurationError):
        P.build_hierarchy(P.random_network(12, 2, seed=0), 4, threshold=1)


def test_random_network_is_bitwise_the_references():
    a = fas.random_network_arrays(32, 5, [3, 32, 5])
    net = P.random_network(32, 5, [3, 32, 5])
    assert np.stack([b.weights for b in net.blocks]).tobytes() == a["W"].tobytes()
    assert np.stack([b.bias for b in net.blocks]).tobytes() == a["b"].tobytes()
    assert net.opening.weights.tobytes() == a["Wo"].tobytes()
    assert net.readout.weights.tobytes() == a["Wr"].tobytes()
    assert net.step_size == a["step"]
    assert np.array_equal(P.random_sample(5, [1, 2]), fas.random_sample(5, [1, 2]))


def test_partition_and_protocol_host_logic():
    part = P.make_partition(32, 4, 3)
    assert part.assignment == [0, 0, 0, 1, 1, 1, 2, 2]
    assert part.cross_edges() == [(2, 3), (5, 6)]
    msg = P.BoundaryMessage(5, np.arange(3.0), 7)
    back = P.decode_message(P.encode_message(msg))
    assert back.sender_block == 5 and back.sweep_tag == 7 and np.array_equal(back.payload, msg.payload)
    with pytest.raises(P.ProtocolError):
        P.decode_message(b"\x00" * 5)
    tr = P.ExchangeTracker()
    tr.check((0, 1), tr.take_tag())
    with pytest.raises(P.ProtocolError):
        tr.check((0, 1), 0)
    with pytest.raises(P.ConfigurationError):
        P.make_partition(10, 4, 1)
