#!/usr/bin/env bash
# round-2 GPU pass: build, tests, bench lines for C1..C5, ncu launch lists and
# --set full captures of the dominant kernels.  Everything lands in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
what="${*:-tests bench lines ncu}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for w in $what; do
  case "$w" in
    tests)
      timeout 3000 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/gpu_tests.log 2>&1
      echo "gpu tests rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests.log | tail -15 ;;
    bench)
      timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
      echo "bench rc=$?"; cat gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err
      timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
      echo "ref rc=$?"; cat gpurun_out/bench_ref.json ;;
    lines)
      for wl in c1 c2 c3 c5; do
        timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
        echo "bench $wl rc=$?"; cat gpurun_out/bench_$wl.json; tail -3 gpurun_out/bench_$wl.err
      done ;;
    ncu)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-check \
        > gpurun_out/bench_c4_under_ncu.log 2>&1
      echo "ncu launches c4 rc=$?"
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
        --log-file gpurun_out/launches_c5.csv python bench.py --workload c5 --steps 1 --warmup 1 --no-cpu-baseline --no-check \
        > gpurun_out/bench_c5_under_ncu.log 2>&1
      echo "ncu launches c5 rc=$?"
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:verify_kernel -c 1 \
        -f -o gpurun_out/prof_verify_c4 python scripts/prof_one.py --span 36 > gpurun_out/prof_c4.log 2>&1
      echo "ncu verify c4 rc=$?"; tail -1 gpurun_out/prof_c4.log
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:sieve_out -c 1 \
        -f -o gpurun_out/prof_sieve_c4 python scripts/prof_one.py --span 34 > gpurun_out/prof_sieve_c4.log 2>&1
      echo "ncu sieve c4 rc=$?"
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:verify_kernel -c 1 \
        -f -o gpurun_out/prof_verify_c5 python scripts/prof_one.py --hi 4000000000000000000 --origin 3999999900000000000 --span 34 > gpurun_out/prof_c5.log 2>&1
      echo "ncu verify c5 rc=$?"; tail -1 gpurun_out/prof_c5.log
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:large_mark -c 1 \
        -f -o gpurun_out/prof_large_c5 python scripts/prof_one.py --hi 4000000000000000000 --origin 3999999900000000000 --span 34 > gpurun_out/prof_large_c5.log 2>&1
      echo "ncu large c5 rc=$?" ;;
    smoke)
      timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
      echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log ;;
  esac
done
