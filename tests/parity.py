"""Helpers comparing the CUDA path (via the C ABI) with the CPU oracle.

Tolerances follow BASELINE.json north_star as made concrete in SURVEY §8(c).4:
integer / index outputs bit-exact; continuous state |x_gpu - x_ref| <=
1e-5 * max(|x_ref|, 1).
"""
import numpy as np

REL = 1e-5

INT_STATE = ("status", "lane", "cursor", "wait_steps", "insert_time", "arrive_time")
JUNC = ("junc_policy", "junc_phase", "junc_elapsed", "junc_yellow_left", "junc_pending",
        "junc_remaining")


def close(a, b, rel=REL):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) <= rel * np.maximum(np.abs(b), 1.0)


def compare_states(g, o, rel=REL, where=""):
    """Bit-exact integer fields, tolerance on s / v (DRIVING vehicles)."""
    for k in INT_STATE:
        bad = np.where(np.asarray(g[k]) != np.asarray(o[k]))[0]
        assert bad.size == 0, f"{where}{k} differs at vids {bad[:10]}: gpu {np.asarray(g[k])[bad[:5]]} oracle {np.asarray(o[k])[bad[:5]]}"
    d = np.asarray(o["status"]) == 1
    for k in ("s", "v"):
        ok = close(np.asarray(g[k])[d], np.asarray(o[k])[d], rel)
        bad = np.where(d)[0][~ok]
        assert bad.size == 0, f"{where}{k} off at vids {bad[:10]}: gpu {np.asarray(g[k])[bad[:5]]} oracle {np.asarray(o[k])[bad[:5]]}"
    for k in JUNC:
        assert np.array_equal(np.asarray(g[k]), np.asarray(o[k])), f"{where}{k}"
    assert np.array_equal(g["lane_signal"][:len(o["lane_signal"])], o["lane_signal"]), f"{where}lane_signal"


def compare_decisions(gd, od, prev_status, rel=REL, where=""):
    drv = np.asarray(prev_status) == 1
    for k in ("leader_vid", "leader_hops", "phantom", "old_follower_vid", "lc", "handoffs",
              "finished"):
        a = np.asarray(gd[k])[drv]
        b = np.asarray(od[k])[drv]
        bad = np.where(drv)[0][a != b]
        assert bad.size == 0, f"{where}{k} differs at vids {bad[:10]}: gpu {np.asarray(gd[k])[bad[:5]]} oracle {np.asarray(od[k])[bad[:5]]}"
    a = np.asarray(gd["side_vid"])[drv]
    b = np.asarray(od["side_vid"])[drv]
    bad = np.where(drv)[0][(a != b).any(axis=1)]
    assert bad.size == 0, f"{where}side_vid differs at vids {bad[:10]}"
    assert np.array_equal(np.asarray(gd["inserted"]) != 0, np.asarray(od["inserted"]) != 0), \
        f"{where}inserted set differs"
    ok = close(np.asarray(gd["accel"])[drv], np.asarray(od["accel"])[drv], rel)
    bad = np.where(drv)[0][~ok]
    assert bad.size == 0, f"{where}accel off at {bad[:10]}: gpu {np.asarray(gd['accel'])[bad[:5]]} oracle {np.asarray(od['accel'])[bad[:5]]}"


def compare_lane_orders(g_off, g_ord, o_off, o_ord, g_state, rel=REL):
    """Per-lane (s, vid) orders: identical except where the swapped vehicles'
    positions are within the continuous tolerance (near-ties, where the order
    is decided by fp rounding; both orders are then valid)."""
    assert np.array_equal(g_off, o_off), "lane counts differ"
    s = np.asarray(g_state["s"], np.float64)
    for l in np.where(np.diff(g_off) > 0)[0]:
        a = g_ord[g_off[l]:g_off[l + 1]]
        b = o_ord[o_off[l]:o_off[l + 1]]
        if np.array_equal(a, b):
            continue
        assert sorted(a) == sorted(b), f"lane {l}: different vehicle sets"
        for x, y in zip(a, b):
            if x != y:
                assert abs(s[x] - s[y]) <= rel * max(abs(s[y]), 1.0), f"lane {l}: order differs beyond ties"
