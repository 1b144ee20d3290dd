#!/bin/bash
# The GPU suite against the alternative step kernel (the warp-specialised ring
# kernel, KS_WARP=0): built as a variant library and put in place of the
# default one for this run only (run on a GPU box; dev tool).
set -e
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p var
bash scripts/build_variant.sh paper_2406_10661_b200/csrc var/lib_ring.so -DKS_WARP=0
cp paper_2406_10661_b200/libsim_b200.so /tmp/libsim_default.so
cp var/lib_ring.so paper_2406_10661_b200/libsim_b200.so && touch paper_2406_10661_b200/libsim_b200.so
python -m pytest tests -m gpu -x -q || rc=$?
cp /tmp/libsim_default.so paper_2406_10661_b200/libsim_b200.so
exit ${rc:-0}
