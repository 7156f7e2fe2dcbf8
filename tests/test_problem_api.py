"""The BAProblem append API of the Python mirror against the reference's own
cases (tests/test_problem.cpp:93-116, 220-232); host-only, no GPU."""
import math

import pytest

import paper_2112_01349_b200 as dba
from paper_2112_01349_b200.dba import CameraState, InvalidArgumentError, Observation, PointState


def test_add_node_append_semantics_and_separate_index_spaces():  # test_problem.cpp:93-102
    p = dba.BAProblem()
    assert p.add_node(CameraState()) == 0
    assert p.add_node(PointState()) == 0
    assert p.add_node(CameraState()) == 1
    with pytest.raises(InvalidArgumentError):
        p.add_node(CameraState(rotation=(math.nan, 0.0, 0.0)))


def test_add_edge_validates_references_and_appends_in_order():  # test_problem.cpp:104-116
    p = dba.BAProblem()
    p.add_node(CameraState())
    p.add_node(PointState())
    assert p.add_edge(Observation()) == 0
    assert p.add_edge(Observation()) == 1
    assert p.num_observations == 2
    with pytest.raises(InvalidArgumentError):
        p.add_edge(Observation(point_id=3))


def test_validate_flags_unreferenced_nodes():  # test_problem.cpp:220-232
    p = dba.BAProblem()
    p.add_node(CameraState())
    p.add_node(CameraState())
    p.add_node(PointState(position=(0.0, 0.0, -1.0)))
    p.add_edge(Observation())
    w = p.validate()
    assert len(w) == 1 and "camera 1" in w[0]
