mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_shard_procs.py -m gpu -q -x -rs > gpurun_out/r2m_pytest.log 2>&1; echo pytest_rc=$?
