#!/usr/bin/env bash
# generic GPU pass: build, then run each argument as a shell command; output under gpurun_out/
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
i=0
for c in "$@"; do
  i=$((i+1))
  echo "== [$i] $c"
  bash -c "$c" 2>&1 | tail -40
  echo "== [$i] rc=${PIPESTATUS[0]}"
done
