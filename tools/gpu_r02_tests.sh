# round-2 GPU parity suite (new tests first), core counts for the oracle timings
set -x
nproc; python -c "import os; print(len(os.sched_getaffinity(0)))"
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 2400 python -m pytest tests/test_gpu_env_cases.py tests/test_gpu_attn_fwd.py tests/test_gpu_index.py tests/test_gpu_configs.py tests/test_gpu_fullsize.py -q -x -s --durations=15 > gpurun_out/r02_pytest_new.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/r02_pytest_new.log
