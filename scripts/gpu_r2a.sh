set -u
cd "${GRAFT_REPO_ROOT}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks_int scripts/micro/peaks_int.cu && timeout 300 /tmp/peaks_int > gpurun_out/peaks_int.json 2>&1; echo "peaks rc=$?"; cat gpurun_out/peaks_int.json
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -25 gpurun_out/gpu_tests.log
