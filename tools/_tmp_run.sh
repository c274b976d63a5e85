mkdir -p gpurun_out
python bench.py --no-cpu > gpurun_out/r3n_bench_chunked.log 2>&1
HG_BIND_ENCRYPT_CHUNKED=0 python bench.py --no-cpu > gpurun_out/r3n_bench_single.log 2>&1
python bench.py --no-cpu > gpurun_out/r3n_bench_chunked2.log 2>&1
HG_BIND_ENCRYPT_CHUNKED=0 python bench.py --no-cpu > gpurun_out/r3n_bench_single2.log 2>&1
timeout 600 python tools/e2e_phases.py c3 > gpurun_out/r3n_phases_chunked.log 2>&1
HG_BIND_ENCRYPT_CHUNKED=0 timeout 600 python tools/e2e_phases.py c3 > gpurun_out/r3n_phases_single.log 2>&1
