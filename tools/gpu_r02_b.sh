# A/B bounds variants + parity report for both grid modes
mkdir -p gpurun_out
bash tools/gpu_ab_short.sh 10 libsmpm.so libsmpm_tight.so
rm -f gpurun_out/parity_r02.jsonl
SMPM_PARITY_REPORT=gpurun_out/parity_r02.jsonl timeout 1500 python -m pytest -q -m gpu tests/test_gpu_configs.py > gpurun_out/pytest_cfg.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_cfg.log
