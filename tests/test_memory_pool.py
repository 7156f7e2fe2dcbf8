"""Predicted-size memory pool: the
host-side prediction of a rank's device footprint (dbag_predict_memory). It
needs no GPU; tests/test_gpu_parity.py::test_memory_pool_matches_prediction
checks that upload reserves exactly this many bytes in one allocation."""
import numpy as np
import pytest

import paper_2112_01349_b200 as dba

ALIGN = 256


@pytest.fixture(scope="module")
def ladybug():
    return dba.generate_synthetic(dba.SyntheticOptions(cameras=49, points=7776, num_observations=31843, seed=1))


LANES = 18  # factored coupling records: G = sqrt(w) Jc per slot (kernels.cuh kLanesFact)


def _floor_bytes(p, k, rank, s, t):
    """Lower bound from the dominant per-edge arrays alone: E records
    (18 lanes of t bytes per slot), the slot arrays (4 int32 + 3 scalars per
    edge). (The fused linearize keeps no per-edge assembly rows; with
    DBAG_LIN=rows they add 28 s per edge, checked below.)"""
    n_k = len(dba.partition_edges(p, k)[rank].edge_ids)
    return n_k * (LANES * t + 16 + 3 * s)


@pytest.mark.parametrize("k", [1, 2, 4])
def test_prediction_bounds_and_split(ladybug, k):
    for rank in range(k):
        b = dba.predict_memory(ladybug, k, rank)
        assert b % ALIGN == 0
        lo = _floor_bytes(ladybug, k, rank, 8, 8)
        assert lo < b < 2 * lo + 4 * 2**20
    # the shards split the edge-proportional part: K ranks together hold
    # about one problem plus the replicated camera space
    tot = sum(dba.predict_memory(ladybug, k, r) for r in range(k))
    one = dba.predict_memory(ladybug, 1, 0)
    assert one <= tot < one * 1.05 + k * 2**20


def test_precision_variants_order(ladybug):
    b64 = dba.predict_memory(ladybug)
    lean = dba.predict_memory(ladybug, coupling_fp32=True)
    p32 = ladybug.astype(np.float32)
    assert lean < b64
    # E lanes dominate the saving: 18 x 4 bytes per slot, up to chunk padding
    n = ladybug.num_observations
    assert LANES * 4 * n <= b64 - lean < LANES * 4 * n * 1.6
    assert dba.predict_memory(p32) < lean


def test_prediction_is_deterministic_and_validates(ladybug):
    assert dba.predict_memory(ladybug, 2, 1) == dba.predict_memory(ladybug, 2, 1)
    with pytest.raises(dba.InvalidArgumentError):
        dba.predict_memory(ladybug, 2, 2)  # rank out of range
    with pytest.raises(dba.InvalidArgumentError):
        dba.predict_memory(ladybug, 0, 0)


def test_assembly_scratch_is_bounded(ladybug, monkeypatch):
    """The Jb assembly rows (28 scalars per edge) are held for one batch of
    whole points at a time (row assembly, DBAG_LIN=rows): with DBAG_JB_BATCH
    slots the pool shrinks by the rows of all but one batch, plus a
    54-double carry per camera."""
    monkeypatch.setenv("DBAG_LIN", "rows")
    full = dba.predict_memory(ladybug)
    monkeypatch.setenv("DBAG_JB_BATCH", "4096")
    small = dba.predict_memory(ladybug)
    n = ladybug.num_observations
    saved = full - small
    assert (n - 4096 - 64) * 28 * 8 - 49 * 54 * 8 - 8 * 2**10 <= saved <= (n - 4096) * 28 * 8 + 4 * 2**10


def test_row_assembly_scratch_in_the_prediction(ladybug, monkeypatch):
    """DBAG_LIN=rows (the two-kernel assembly through per-edge Jacobian rows)
    adds its 28 scalars per edge of row scratch to the pool, and the fused
    path's 54-double camera partials are gone from it."""
    fused = dba.predict_memory(ladybug)
    monkeypatch.setenv("DBAG_LIN", "rows")
    rows = dba.predict_memory(ladybug)
    n = ladybug.num_observations
    assert 28 * 8 * n * 0.6 < rows - fused < 33 * 8 * n  # + camera-major slot lists (4 B per edge)
