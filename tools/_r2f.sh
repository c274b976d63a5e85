mkdir -p gpurun_out
for cfg in c3 c5; do
  timeout 600 python tools/diag_step.py $cfg 8 > gpurun_out/r2f_diag_${cfg}_tc1.log 2>&1
  HG_GEMM_TC=0 timeout 600 python tools/diag_step.py $cfg 8 > gpurun_out/r2f_diag_${cfg}_tc0.log 2>&1
done
timeout 900 python tools/diag_step.py c4 6 > gpurun_out/r2f_diag_c4.log 2>&1
python bench.py --config c5 --batch 8192 --no-cpu > gpurun_out/r2f_bench_c5.log 2>&1; echo c5_rc=$?
python bench.py --config c4 --batch 8192 --steps 5 --warmup 3 --no-cpu > gpurun_out/r2f_bench_c4.log 2>&1; echo c4_rc=$?
