# gpurun -- bash tools/gpu_suite_and_evidence.sh: the full GPU suite, then the round-2 evidence run
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/s4_pytest.log
tail -30 gpurun_out/s4_pytest.log
bash tools/evidence_r2.sh > gpurun_out/s4_evidence.log 2>&1
tail -c 2500 gpurun_out/bench_r2.log
