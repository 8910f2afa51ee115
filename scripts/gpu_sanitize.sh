#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over every libgb
# kernel (scripts/sanitize_driver.py: small invocations, each an oracle parity check)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for t in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$t" = racecheck ] && extra="--racecheck-report all"
  timeout 2400 compute-sanitizer --tool $t $extra --print-limit 20 python scripts/sanitize_driver.py \
    > gpurun_out/r02_$t.log 2>&1
  echo "$t rc=$?"; tail -3 gpurun_out/r02_$t.log
done
