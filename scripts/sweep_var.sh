#!/bin/bash
# time every var/lib_*.so on C4 (dev tool; PREROLL=200)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PREROLL=${PREROLL:-200}
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 120 python scripts/time_c4.py 2>&1 | head -1
for f in var/lib_*.so; do timeout 120 python scripts/time_c4.py $f 2>&1 | head -1; done
