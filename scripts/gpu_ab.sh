#!/usr/bin/env bash
# A/B pass on the GPU box: every ab/*.so against the default libgb.so on the top 2^36
# integers of [4, 1e12] (C4) and of the C5 window (scripts/ab_time.py; result digests
# must agree), plus the L2 RED-rate-vs-SM-count microbenchmark.  Output in gpurun_out/.
#   bash scripts/gpu_ab.sh [c4] [c5] [sieve] [micro]
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
what="${*:-c4 c5 micro}"
for w in $what; do
  case "$w" in
    c4) timeout 1200 python scripts/ab_time.py --abdir ${ABDIR:-ab} --span 36 --reps 10 --rounds 2 > gpurun_out/ab_c4.log 2>&1
        echo "ab c4 rc=$?"; cat gpurun_out/ab_c4.log | cut -c1-260 ;;
    c5) timeout 1500 python scripts/ab_time.py --abdir ${ABDIR:-ab} --span 36 --reps 5 --rounds 2 --hi 4000000000000000000 > gpurun_out/ab_c5.log 2>&1
        echo "ab c5 rc=$?"; cat gpurun_out/ab_c5.log | cut -c1-260 ;;
    sieve) for lib in paper_2603_02621_b200/libgb.so ${ABDIR:-ab}/*.so paper_2603_02621_b200/libgb.so ${ABDIR:-ab}/*.so; do
             for N in 1e12 4e18; do GB_LIB=$PWD/$lib timeout 300 python scripts/sieve_time.py --N $N 2>&1 | tail -1; done
           done > gpurun_out/ab_sieve.log 2>&1
        echo "ab sieve rc=$?"; cat gpurun_out/ab_sieve.log ;;
    micro) nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/red_sms scripts/micro/red_sms.cu \
             && timeout 300 /tmp/red_sms > gpurun_out/red_sms.json 2>&1
        echo "red_sms rc=$?"; cat gpurun_out/red_sms.json ;;
  esac
done
