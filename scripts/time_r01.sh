#!/bin/bash
# The round-1 step kernel (commit 3998616) on the bench's current workload (C4,
# 200-step pre-roll, L2 flush before each timed step), for a before / after on
# the same input: builds the r01 library from git into var/r01 and times it
# with the r01 Python binding.  Dev tool (run on a GPU box).
set -e
cd "${GRAFT_REPO_ROOT:-/root/repo}"
if [ ! -f var/r01/paper_2406_10661_b200/libsim_b200.so ]; then
  rm -rf var/r01 && mkdir -p var/r01
  git archive 3998616 paper_2406_10661_b200 include | tar -x -C var/r01
  (cd var/r01 && /usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a \
     -Xcompiler -fPIC -shared -Iinclude -Ipaper_2406_10661_b200/csrc \
     -o paper_2406_10661_b200/libsim_b200.so paper_2406_10661_b200/csrc/kernels.cu \
     paper_2406_10661_b200/csrc/sim_api.cu)
fi
python - <<'PY'
import os, sys
root = os.getcwd()
sys.path.insert(0, os.path.join(root, "var", "r01"))   # the r01 package first
sys.path.insert(1, root)                               # synth (C4 recipe unchanged since r01)
import numpy as np, torch, synth
import paper_2406_10661_b200.sim as S
assert "var/r01" in S.__file__, S.__file__
cache = "/tmp/c4.npz"
scen = synth.load_scenario(cache) if os.path.exists(cache) else synth.city()
st = torch.cuda.Stream()
sim = S.Sim.from_scenario(scen, stream=st.cuda_stream)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sim.step(int(os.environ.get("PREROLL", "200"))); sim.sync()
sim.enable_timing(True)
n = 40
m0 = sim.read_metrics()
with torch.cuda.stream(st):
    for k in range(n):
        flush.fill_(k & 255)
        sim.step(1)
torch.cuda.synchronize()
ks, sg, nl = sim.read_timing()
m1 = sim.read_metrics()
vs = m1["vehicle_steps"] - m0["vehicle_steps"]
print(f"r01 build (3998616): k_step {ks/n*1e3:.1f} us  k_signal {sg/n*1e3:.1f} us  "
      f"veh-steps/s(kstep) {vs/(ks/1e3):.3e}  lc/step {(m1['n_lane_changes']-m0['n_lane_changes'])/n:.0f}  "
      f"handoffs/step {(m1['n_handoffs']-m0['n_handoffs'])/n:.0f}", flush=True)
PY
