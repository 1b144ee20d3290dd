"""A short run of the hot path for compute-sanitizer (VERDICT r01
#10): C1 ring and a small C2-shaped grid (incl. lane changes, hand-offs,
insertions, MAX_PRESSURE) for a few eager steps and two step-graph replays,
plus the read-side kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2406_10661_b200 as p  # noqa: E402

for scen in (synth.ring(), synth.grid(rows=3, cols=3, road_len=200.0, lanes=2, n_trips=600,
                                     seed=7, depart_window=40, policy=synth.POLICY_MAXP)):
    g = p.Sim.from_scenario(scen)
    g.step(int(os.environ.get("SAN_STEPS", "6")))
    g.step(12)                                      # a step-graph replay pair (PDL, t_base)
    m = g.read_metrics(lane_stats=True)
    st = g.read_state(lane_order=True)
    print(scen.name, m["vehicle_steps"], m["n_handoffs"], m["n_inserted"], flush=True)
