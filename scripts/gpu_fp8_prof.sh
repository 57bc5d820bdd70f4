cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/fp8_prof.py || exit 1
B="python scripts/fp8_prof.py"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_fp8_c2.csv $B > /dev/null 2>&1; echo launches rc=$?
cap() {
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:$2" -s $3 -c 1 -o gpurun_out/prof_$1 $B > gpurun_out/ncu_$1.log 2>&1; echo $1 rc=$?
}
cap f8_spmm_fwdout 'EpiStoreI13__nv_bfloat16Lb1E' 2
cap f8_k1 'EpiFwd1TILb1E' 1
cap f8_spmm_dw 'EpiStoreIfLb1E' 2
cap f8_quant_rows 'k_quant_rows' 10
for f in f8_spmm_fwdout f8_k1 f8_spmm_dw f8_quant_rows; do python scripts/ncu_summary.py gpurun_out/prof_$f.ncu-rep > gpurun_out/ncu_$f.txt 2>&1; done
cuobjdump -sass paper_2503_16672_b200/libs24.so 2>/dev/null | grep -o "UTC[A-Z0-9_.]*MMA[A-Z0-9_.]*" | sort | uniq -c > gpurun_out/sass_mma_ops.txt
