set -x
python bench.py > gpurun_out/bench8.log 2> gpurun_out/bench8.err; echo bench_rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref8.log 2>&1; echo ref_rc=$?
timeout 600 python tools/prim_sweep.py --out gpurun_out/sweep8.jsonl > gpurun_out/sweep8.log 2>&1; echo sweep_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches8.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu8a.log 2>&1; echo ncua_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_relin_t|k_rescale_rest_t|k_encrypt_t|k_gemm_tc" -s 0 -c 4 -o gpurun_out/full8 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu8b.log 2>&1; echo ncub_rc=$?
