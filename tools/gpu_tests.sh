# GPU tests + smoke (run under gpurun); parity report lines -> gpurun_out/parity_r02.jsonl
mkdir -p gpurun_out
rm -f gpurun_out/parity_r02.jsonl
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
SMPM_PARITY_REPORT=gpurun_out/parity_r02.jsonl timeout 1500 python -m pytest -m gpu -q -s ${PYTEST_ARGS:-tests} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -n 5 gpurun_out/smoke.log gpurun_out/pytest_gpu.log
