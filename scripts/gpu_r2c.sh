#!/usr/bin/env bash
# round-2 measurement pass: build, smoke, the GPU tests, bench lines (C1..C5, the
# reference arm, the comparison modes and NEXT-4 counts), ncu launch lists and
# --set full captures of every dominant kernel.  Everything lands in gpurun_out/.
#   bash scripts/gpu_r2c.sh [tests] [bench] [lines] [modes] [ncu]
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
what="${*:-tests bench lines modes ncu}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
B="timeout 900 python bench.py"
for w in $what; do
  case "$w" in
    tests)
      timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
      echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
      timeout 3000 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/gpu_tests.log 2>&1
      echo "gpu tests rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests.log | tail -15 ;;
    bench)
      $B --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
      echo "bench rc=$?"; cut -c1-400 gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err
      $B --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
      echo "ref rc=$?"; cut -c1-300 gpurun_out/bench_ref.json ;;
    lines)
      for wl in c1 c2 c3 c5; do
        $B --workload $wl --steps 5 --warmup 3 > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err
        echo "bench $wl rc=$?"; cut -c1-300 gpurun_out/bench_$wl.json; tail -2 gpurun_out/bench_$wl.err
      done
      $B --N 1e13 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n1e13.json 2> gpurun_out/bench_n1e13.err
      echo "bench 1e13 rc=$?"; cut -c1-300 gpurun_out/bench_n1e13.json ;;
    modes)
      $B --mode counts --steps 5 --warmup 3 > gpurun_out/bench_counts.json 2> gpurun_out/bench_counts.err
      echo "counts rc=$?"; cut -c1-400 gpurun_out/bench_counts.json; tail -2 gpurun_out/bench_counts.err
      $B --workload c3 --mode pern --steps 3 --warmup 3 --no-cpu-baseline --no-sieve > gpurun_out/bench_c3_pern.json 2> gpurun_out/bench_c3_pern.err
      echo "pern rc=$?"; cut -c1-300 gpurun_out/bench_c3_pern.json
      $B --workload c3 --mode resident --steps 3 --warmup 3 --no-cpu-baseline --no-sieve > gpurun_out/bench_c3_resident.json 2> gpurun_out/bench_c3_resident.err
      echo "resident rc=$?"; cut -c1-300 gpurun_out/bench_c3_resident.json ;;
    ncu)
      N="timeout 900 ncu --clock-control none"
      $N --metrics gpu__time_duration.sum -c 400 --csv --log-file gpurun_out/launches_c4.csv \
        python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-check > /dev/null 2>&1
      echo "ncu launches c4 rc=$?"
      $N --metrics gpu__time_duration.sum -c 2000 --csv --log-file gpurun_out/launches_c5.csv \
        python bench.py --workload c5 --steps 1 --warmup 1 --no-cpu-baseline --no-check > /dev/null 2>&1
      echo "ncu launches c5 rc=$?"
      F="$N --set full --import-source on -c 1 -f"
      S="python scripts/ncu_summary.py"
      # each capture is summarised here (ncu -i works on the box) and only the C4
      # verify report is kept: gpurun copies back at most 64 MiB
      $F -k regex:verify_kernel -o gpurun_out/prof_verify_c4 python scripts/prof_one.py --span 36 > gpurun_out/prof_c4.log 2>&1
      echo "ncu verify c4 rc=$?"
      python scripts/ncu_regions.py gpurun_out/prof_verify_c4.ncu-rep > gpurun_out/regions_verify_c4.txt 2>&1
      $S gpurun_out/prof_verify_c4.ncu-rep gpurun_out/sum_verify_kernel_c4 --evens 34359738368 \
        --note "ncu --set full --clock-control none, one gb_verify_range over the top 2^36 integers of [4, 1e12] (scripts/prof_one.py --span 36)" > /dev/null
      $F -k regex:sieve_out -o gpurun_out/prof_sieve_c4 python scripts/prof_one.py --span 34 > /dev/null 2>&1
      echo "ncu sieve c4 rc=$?"
      $S gpurun_out/prof_sieve_c4.ncu-rep gpurun_out/sum_sieve_out_kernel_c4 --evens 8589934592 \
        --note "ncu --set full, gb_sieve_segment (sieve_out_kernel) over the top 2^34 integers of [4, 1e12] (evens = integers / 2)" > /dev/null
      rm -f gpurun_out/prof_sieve_c4.ncu-rep
      $F -k regex:verify_kernel -o gpurun_out/prof_verify_c5 python scripts/prof_one.py --hi 4000000000000000000 --span 34 > /dev/null 2>&1
      echo "ncu verify c5 rc=$?"
      $S gpurun_out/prof_verify_c5.ncu-rep gpurun_out/sum_verify_kernel_c5 --evens 872939520 \
        --note "ncu --set full, the first verify launch (one K-LARGE chunk: 444 tiles = 8.73e8 evens) of the top 2^34 integers of [4e18 - 1e11, 4e18)" > /dev/null
      python scripts/ncu_regions.py gpurun_out/prof_verify_c5.ncu-rep > gpurun_out/regions_verify_c5.txt 2>&1
      rm -f gpurun_out/prof_verify_c5.ncu-rep
      $F -k regex:large_mark -o gpurun_out/prof_large_c5 python scripts/prof_one.py --hi 4000000000000000000 --span 34 > /dev/null 2>&1
      echo "ncu large c5 rc=$?"
      $S gpurun_out/prof_large_c5.ncu-rep gpurun_out/sum_large_mark_wheel_kernel_c5 --evens 872939520 \
        --note "ncu --set full, the first K-LARGE mark launch (one chunk: 444 tiles = 8.73e8 evens) of the top 2^34 integers of the C5 window" > /dev/null
      rm -f gpurun_out/prof_large_c5.ncu-rep
      $F -k regex:counts_kernel -o gpurun_out/prof_counts python bench.py --mode counts --steps 1 --warmup 1 --no-check > /dev/null 2>&1
      echo "ncu counts rc=$?"
      $S gpurun_out/prof_counts.ncu-rep gpurun_out/sum_counts_kernel_counts --evens 16384 \
        --note "ncu --set full, gb_partition_counts of the top 16384 even n below 1e9 (bench.py --mode counts)" > /dev/null
      rm -f gpurun_out/prof_counts.ncu-rep
      ls -la gpurun_out | tail -30 ;;
  esac
done
