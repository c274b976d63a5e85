set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t11.log 2>&1; echo t_rc=$?
cap() {  # name regex skip
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$2" -s "$3" -c 1 -o /tmp/$1 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_$1.log 2>&1
  python tools/ncu_to_profile.py /tmp/$1.ncu-rep "$4" gpurun_out/$1 > /dev/null 2>&1
  python tools/ncu_lines.py /tmp/$1.ncu-rep "" 30 > gpurun_out/$1_lines.txt 2>&1
  rm -f /tmp/$1.ncu-rep
}
cap r1_ncu_relin_u32 k_relin_t 0 k_relin_t/u32
cap r1_ncu_relin_f64 k_relin_t 1 k_relin_t/f64
cap r1_ncu_rescale_u32 k_rescale_rest_t 0 k_rescale_rest_t/u32
cap r1_ncu_encrypt_u32 k_encrypt_t 0 k_encrypt_t/u32
timeout 600 python tools/prim_sweep.py --ns 8192 --ls 7 > gpurun_out/sweep11.log 2>&1
du -sh gpurun_out/*
