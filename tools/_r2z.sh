mkdir -p gpurun_out
cap() {  # name kernel-regex launches-to-skip traffic-key workload-command...
  local name=$1 rx=$2 skip=$3 key=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s "$skip" -c 1 \
    -o /tmp/$name "$@" > gpurun_out/ncu_$name.log 2>&1
  python tools/ncu_to_profile.py /tmp/$name.ncu-rep "$key" gpurun_out/$name > /dev/null 2>&1
  python tools/ncu_lines.py /tmp/$name.ncu-rep "" 40 > gpurun_out/${name}_lines.txt 2>&1
  rm -f /tmp/$name.ncu-rep
}
export ITERS=1
cap r2z_ncu_encrypt_a k_encrypt 0 k_encrypt_a python tools/e2e_breakdown.py c3
cap r2z_ncu_encrypt_b k_encrypt 1 k_encrypt_b python tools/e2e_breakdown.py c3
cap r2z_ncu_sample k_sample_encryption 0 k_sample python tools/e2e_breakdown.py c3
HG_ENCRYPT_PIPE=1 ITERS=5 python tools/e2e_breakdown.py c3 > gpurun_out/r2z_e2e_pipe.log 2>&1
