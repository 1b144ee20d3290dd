"""Mutation check of the oracle's rule pins (VERDICT r01 "Next round" #1).

For each rule the oracle follows (ledger readings), apply one
plausible mistake to a COPY of oracle/oracle.cpp, build it into /tmp, and run
tests/test_oracle_rule_pins.py + tests/test_oracle_pins.py against it
(ORACLE_LIB_OVERRIDE).  A mutation that leaves every pin green is reported as
SURVIVED (a gap in the pins).  Writes profiles/r02_oracle_mutations.txt.

    python scripts/oracle_mutations.py
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.cpp")

# (name, rule, original text, mutated text)
MUTATIONS = [
    ("ins-ahead-sign", "O10 ahead gap (L25)",
     "((V[ahead].s - me.start_s) - veh_len(ahead)) >= p.s0",
     "((me.start_s - V[ahead].s) - veh_len(ahead)) >= p.s0"),
    ("ins-ahead-strict", "O10 ahead gap >= (L25)",
     "((V[ahead].s - me.start_s) - veh_len(ahead)) >= p.s0",
     "((V[ahead].s - me.start_s) - veh_len(ahead)) > p.s0"),
    ("ins-behind-sign", "O10 behind gap (L25)",
     "((me.start_s - V[behind].s) - p.len) >= need",
     "((V[behind].s - me.start_s) - p.len) >= need"),
    ("ins-behind-no-vb", "O10 behind one-step advance (L25)",
     "double need = (V[behind].v + 0.5 * pb.a_max) + p.s0;",
     "double need = (0.5 * pb.a_max) + p.s0;"),
    ("ins-behind-ego-amax", "O10 behind vehicle's a_max (L25)",
     "double need = (V[behind].v + 0.5 * pb.a_max) + p.s0;",
     "double need = (V[behind].v + 0.5 * p.a_max) + p.s0;"),
    ("ins-behind-len", "O10 inserted vehicle's length (L25)",
     "((me.start_s - V[behind].s) - p.len) >= need",
     "((me.start_s - V[behind].s) - pb.len) >= need"),
    ("ins-no-margin", "O10 lane-start margin (L17/L25)",
     "if (!((me.start_s - p.len) >= start_margin)) return false;",
     "if (!((me.start_s - p.len) >= 0.0)) return false;"),
    ("ins-priority-vid", "O10 (depart, vid) priority (L25)",
     "if (V[a].depart != V[b].depart) return V[a].depart < V[b].depart;\n        return a < b;",
     "return a < b;"),
    ("ins-tie-desc", "O10 ties by vid (L25)",
     "if (V[a].depart != V[b].depart) return V[a].depart < V[b].depart;\n        return a < b;",
     "if (V[a].depart != V[b].depart) return V[a].depart < V[b].depart;\n        return a > b;"),
    ("ins-many-per-lane", "O10 one insertion per lane per step (L25)",
     "if (insertion_ok(k, l, order[l])) { inserted.push_back(k); pend_head[l]++; }",
     "while (pend_head[l] < pend[l].size() && V[pend[l][pend_head[l]]].depart <= t &&\n"
     "             insertion_ok(pend[l][pend_head[l]], l, order[l])) {\n"
     "        inserted.push_back(pend[l][pend_head[l]]); pend_head[l]++; }"),
    ("mand-swap", "mandatory side LEFT/RIGHT (L18/L37)",
     "mand = left_ok ? -1 : (right_ok ? +1 : 0);",
     "mand = left_ok ? +1 : (right_ok ? -1 : 0);"),
    ("mand-right-first", "mandatory side preference (L37)",
     "mand = left_ok ? -1 : (right_ok ? +1 : 0);",
     "mand = right_ok ? +1 : (left_ok ? -1 : 0);"),
    ("mand-draw", "mandatory change without a draw (L18)",
     "if (adm[sd]) choice = sd;                            // L18",
     "if (adm[sd] && u53(seed, k, t) < p_lc(std::max(0.0, u[sd]))) choice = sd;"),
    ("stopline-dropped", "lane end is a stop line outside G (L18, P:200)",
     "(e.next1 == LANE_BLOCKED || (!is_road(e.next1) && sig[e.next1] != SIG_GREEN))",
     "(e.next1 >= 0 && !is_road(e.next1) && sig[e.next1] != SIG_GREEN)"),
    ("exit-lowest-only", "junction-lane choice (L24)",
     "return best_pref >= 0 ? best_pref : best_any;",
     "return best_any;"),
    ("exit-no-fallback", "junction-lane choice fallback (L24)",
     "return best_pref >= 0 ? best_pref : best_any;",
     "return best_pref >= 0 ? best_pref : LANE_BLOCKED;"),
    ("look-no-Lm", "lookahead gap adds the skipped lane's length (P:168-169)",
     "        d = d + L[m];\n",
     "        d = d + 0.0;\n"),
    ("look-no-len", "lookahead gap subtracts the leader's length (L3)",
     "e.gap = (d + V[f].s) - veh_len(f);",
     "e.gap = (d + V[f].s);"),
    ("stop-branch", "integrator in-step stop (L1)",
     "if (vr < 0.0) { s1 = me.s - ((me.v * me.v) / (2.0 * a)); v1 = 0.0; }",
     "if (vr < 0.0) { s1 = me.s + ((me.v + vr) * 0.5); v1 = 0.0; }"),
    ("one-handoff", "several lanes in one step (L31)",
     "        n = is_road(curl) ? next_from_road(curl, me, ri) : succ[curl][0];\n        continue;",
     "        n = is_road(curl) ? next_from_road(curl, me, ri) : succ[curl][0];\n        break;"),
]


def main():
    src = open(SRC).read()
    out, survived = [], 0
    tmp = tempfile.mkdtemp(prefix="ormut_")
    for name, rule, a, b in MUTATIONS:
        if src.count(a) != 1:
            out.append(f"{name:22s} ERROR: pattern found {src.count(a)} times")
            continue
        cpp = os.path.join(tmp, f"{name}.cpp")
        lib = os.path.join(tmp, f"{name}.so")
        open(cpp, "w").write(src.replace(a, b))
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-I", os.path.join(ROOT, "oracle"), "-o", lib, cpp])
        env = dict(os.environ, ORACLE_LIB_OVERRIDE=lib)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                            "tests/test_oracle_rule_pins.py", "tests/test_oracle_pins.py"],
                           cwd=ROOT, env=env, capture_output=True, text=True)
        failed = [ln.split(" - ")[0].replace("FAILED ", "") for ln in r.stdout.splitlines()
                  if ln.startswith("FAILED")]
        if r.returncode == 0:
            survived += 1
            out.append(f"{name:22s} SURVIVED  ({rule})")
        else:
            out.append(f"{name:22s} killed by {failed[0] if failed else '?'}  ({rule})")
    out.append(f"{len(MUTATIONS) - survived}/{len(MUTATIONS)} mutations killed")
    text = "\n".join(out)
    print(text)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "r02_oracle_mutations.txt"), "w") as f:
        f.write("# scripts/oracle_mutations.py: one plausible mistake per rule applied to a copy of\n"
                "# oracle/oracle.cpp; the pins (tests/test_oracle_rule_pins.py, test_oracle_pins.py)\n"
                "# must fail for each.\n" + text + "\n")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main())
