#!/bin/bash
# The GPU suite against the bounds-checked build (ST_CHECK traps on a row index
# outside its tensor; DESIGN.md §7 "Memory safety without compute-sanitizer").
#   bash scripts/checked_suite.sh <outdir> [pytest args...]
out=${1:-gpurun_out/checked}
shift
mkdir -p "$out"
python -m paper_2410_20790_b200.build --checked > "$out/build.log" 2>&1 || { tail -30 "$out/build.log"; exit 1; }
ST_LIB=$(pwd)/paper_2410_20790_b200/libsparsetem_checked.so ST_NO_GRAPHS=1 \
  timeout ${CHECK_TIMEOUT:-2400} python -m pytest tests -m gpu -q -p no:cacheprovider "$@" > "$out/pytest.log" 2>&1
rc=$?
echo "checked suite rc=$rc: $(tail -1 "$out/pytest.log"); ST_CHECK failures: $(grep -c 'ST_CHECK failed' "$out/pytest.log")" | tee "$out/summary.txt"
