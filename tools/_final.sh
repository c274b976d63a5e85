python bench.py > gpurun_out/bench_f.log 2> gpurun_out/bench_f.err; echo bench_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_f.csv python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_tc -s 0 -c 1 -o /tmp/gtc python tools/diag_step.py c5 > /dev/null 2>&1
python tools/ncu_to_profile.py /tmp/gtc.ncu-rep k_gemm_tc_c5 gpurun_out/r1_ncu_gemm_tc_c5 > /dev/null 2>&1
python tools/ncu_lines.py /tmp/gtc.ncu-rep "" 30 > gpurun_out/r1_ncu_gemm_tc_c5_lines.txt 2>&1
rm -f /tmp/gtc.ncu-rep
timeout 600 python tools/diag_step.py c5 > gpurun_out/diag_c5_f.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_f.log 2>&1; echo t_rc=$?
