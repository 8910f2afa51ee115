#!/usr/bin/env bash
# One gpurun call's worth of GPU work: build, GPU parity tests, bench (both arms),
# the ncu launch list of the bench command and one `ncu --set full` capture of the
# verify kernel.  Everything lands in gpurun_out/.
#   gpurun --timeout 3000 -- 'bash scripts/gpu_round.sh [tests|bench|ncu ...]'
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
what="${*:-tests bench ncu}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/smi.txt 2>&1
for w in $what; do
  case "$w" in
    tests)
      timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
      echo "gpu tests rc=$?"; tail -3 gpurun_out/gpu_tests.log ;;
    smoke)
      timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
      echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log ;;
    bench)
      timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
      echo "bench rc=$?"; cat gpurun_out/bench.json
      timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
      echo "ref rc=$?"; cat gpurun_out/bench_ref.json ;;
    ncu)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
        > gpurun_out/bench_under_ncu.log 2>&1
      echo "ncu launches rc=$?"
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:verify_kernel -c 1 \
        -f -o gpurun_out/prof python scripts/prof_one.py --span 36 > gpurun_out/prof.log 2>&1
      echo "ncu full rc=$?"; tail -2 gpurun_out/prof.log ;;
    t4e18)
      timeout 1200 python -m pytest tests/test_gpu_4e18.py -x -q > gpurun_out/gpu_tests_4e18.log 2>&1
      echo "4e18 tests rc=$?"; tail -3 gpurun_out/gpu_tests_4e18.log ;;
    c5)
      timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
      echo "bench c5 rc=$?"; cat gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
        --log-file gpurun_out/launches_c5.csv python bench.py --workload c5 --steps 1 --warmup 1 --no-cpu-baseline \
        > gpurun_out/bench_c5_under_ncu.log 2>&1
      echo "ncu c5 launches rc=$?" ;;
    sanitize)
      for tool in memcheck racecheck synccheck initcheck; do
        timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_driver.py \
          > gpurun_out/sanitize_$tool.log 2>&1
        echo "sanitize $tool rc=$?"; tail -2 gpurun_out/sanitize_$tool.log
      done ;;
    time)
      timeout 600 python scripts/prof_one.py --span 36 --time 10 2>&1 | tail -2 ;;
  esac
done
