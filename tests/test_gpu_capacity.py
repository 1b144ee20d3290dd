"""Capacity handling of the tile record regions (VERDICT r01 "Next round" #3,
ADVICE r01): a road tile holds at most `cap` stayers (jam
capacity x 1.25 + 16).  Overlapping states (L32) can push a tile past it; the
step kernel must then flag the overflow (sticky SIM_E_CAPACITY at the next
synchronising call) instead of writing into the next tile's records."""
import numpy as np
import pytest

from synth import NetBuilder, Scenario, default_profiles, default_params
from synth.networks import POLICY_NONE, TURN_STRAIGHT

import pin_scenarios as PS

pytestmark = pytest.mark.gpu
SIM_E_CAPACITY = 7


@pytest.fixture(scope="module")
def simlib():
    import paper_2406_10661_b200 as p
    p.build()
    return p


def _cap(L, lmin=5.0):
    """c = floor(L / shortest vehicle) + 2 per lane; cap = (c + c/4 + 16) rounded up to 4."""
    c = int(np.floor(L / lmin)) + 2
    return (c + c // 4 + 16 + 3) & ~3


def _scenario(n_b, n_feed):
    """Road A (4 lanes, 100 m) -> junction -> road B (1 lane, 200 m, dead end).
    n_b vehicles at rest, overlapping, at s in [10, 20] of B; on each lane of A
    n_feed vehicles (v = 10, 6 m apart) heading into B."""
    b = NetBuilder()
    A = b.add_road(4, 100.0, PS.VMAX)
    B = b.add_road(1, 200.0, PS.VMAX)
    J = b.add_junction(policy=POLICY_NONE)
    for a in b.road_lanes[A]:
        b.connect(J, a, b.road_lanes[B][0], TURN_STRAIGHT, 20.0, PS.VMAX)
    rows = [dict(route=[B], lane=b.road_lanes[B][0], s=10.0 + 10.0 * k / max(n_b, 1), v=0.0, end_s=200.0)
            for k in range(n_b)]
    for a in b.road_lanes[A]:
        rows += [dict(route=[A, B], lane=a, s=99.0 - 6.0 * k, v=10.0, end_s=200.0) for k in range(n_feed)]
    return Scenario("cap", b.graph(), PS.trips(rows), default_profiles(), default_params(5))


def test_load_beyond_capacity_is_refused(simlib):
    cap = _cap(200.0)
    simlib.Sim.from_scenario(_scenario(cap, 0))            # exactly full: accepted
    with pytest.raises(simlib.SimError) as e:
        simlib.Sim.from_scenario(_scenario(cap + 1, 0))
    assert e.value.status == SIM_E_CAPACITY


def test_step_overflow_is_flagged(simlib):
    """A full tile B receiving entrants from four junction lanes: its stayers
    exceed the record region, and the handle reports SIM_E_CAPACITY."""
    cap = _cap(200.0)
    g = simlib.Sim.from_scenario(_scenario(cap, 6))
    m = g.read_metrics()
    assert m["n_driving"] == cap + 24
    raised = None
    for _ in range(12):
        g.step(1)
        try:
            g.read_metrics()
        except simlib.SimError as e:
            raised = e
            break
    assert raised is not None and raised.status == SIM_E_CAPACITY
    with pytest.raises(simlib.SimError):                    # sticky
        g.step(1)
        g.sync()


def test_no_overflow_below_capacity(simlib, oracle_lib):
    """The same inflow into a tile with room to spare: no flag, and the state
    agrees with the oracle (exact mode, bit for bit)."""
    cap = _cap(200.0)
    scen = _scenario(cap - 40, 6)
    g = simlib.Sim.from_scenario(scen, exact_mode=True)
    o = oracle_lib.Oracle(scen, store_fp32=True)
    g.step(12)
    o.step(12)
    gs, os_ = g.read_state(), o.read_state()
    for k in ("status", "lane", "cursor", "wait_steps"):
        assert np.array_equal(gs[k], os_[k]), k
    d = os_["status"] == 1
    assert np.array_equal(gs["s"][d].astype(np.float64), os_["s"][d])
    assert g.read_metrics()["n_handoffs"] > 0
