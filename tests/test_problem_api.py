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


def test_check_convergence_decisions():  # tests/test_solver.cpp:457-486
    cfg = dba.SolverConfig(max_iterations=50)
    st = dba.SolverState(x_c=None, x_p=None, lambda_=1e-4, nu=2.0, iteration=3, cost=10.0, termination="",
                         history=[], previous_cost=10.0)
    st.last_accepted, st.last_cost_change, st.last_step_inf = True, 0.0, 1.0
    assert dba.check_convergence(st, cfg) == "converged"
    st.last_cost_change = 5.0
    assert dba.check_convergence(st, cfg) == "keep_going"
    st.last_step_inf = 1e-9
    assert dba.check_convergence(st, cfg) == "converged"
    st.last_accepted, st.last_step_inf, st.iteration = False, 1.0, 50
    assert dba.check_convergence(st, cfg) == "max_iterations"
    st.iteration, st.lambda_ = 3, 2e32
    assert dba.check_convergence(st, cfg) == "stalled"


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [dict(max_iterations=3), dict(max_iterations=50, pcg_tol=1e-10)])
def test_returned_state_decides_its_termination(cfg):
    """The state lm_solve returns carries the last trial (dba/solver.hpp:80-84):
    check_convergence on it gives the solve's own termination reason."""
    p = dba.generate_synthetic(dba.SyntheticOptions(cameras=24, points=200, obs_per_point=6, seed=2024,
                                                    circle_radius=1.0, pixel_noise=0.5))
    c = dba.SolverConfig(**cfg)
    st = dba.lm_solve(p, c)
    assert st.last_accepted == st.history[-1].accepted
    assert dba.check_convergence(st, c) == st.termination


def test_accessors_and_pack_unpack_round_trip():  # dba/problem.hpp:219-227, 294-353
    from tests.factory import ProblemFactory
    p = ProblemFactory(7).random_problem(3, 5, 9)
    cams, pts, cid, pid, px, py, w = p.arrays()
    assert p.camera(1).params() == list(cams[1]) and list(p.point(4).position) == list(pts[4])
    o = p.observation(8)
    assert (o.camera_id, o.point_id, o.pixel, o.weight) == (cid[8], pid[8], (px[8], py[8]), w[8])
    assert len(p.cameras()) == 3 and len(p.points()) == 5 and len(p.observations()) == 9
    xc, xp = dba.pack_cameras(p), dba.pack_points(p)
    dba.unpack_states(xc + 1.0, xp - 2.0, p)
    assert (dba.pack_cameras(p) == xc + 1.0).all() and (dba.pack_points(p) == xp - 2.0).all()
    with pytest.raises(dba.dba.ShapeError):
        dba.unpack_states(xc[:-1], xp, p)
