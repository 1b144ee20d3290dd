#!/bin/bash
# test_variant.sh <variant .so> [pytest args...]: the GPU tests against a
# variant library put in place of the default one for this run (dev tool).
set -e
cd "${GRAFT_REPO_ROOT:-/root/repo}"
lib=$1; shift
cp paper_2406_10661_b200/libsim_b200.so /tmp/libsim_default.so
cp "$lib" paper_2406_10661_b200/libsim_b200.so
touch paper_2406_10661_b200/libsim_b200.so
python -m pytest "$@" || rc=$?
cp /tmp/libsim_default.so paper_2406_10661_b200/libsim_b200.so
exit ${rc:-0}
