# Round profiles: launch list of the bench command + full captures of the top kernels
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-dense"
timeout 300 $B > gpurun_out/prof_plain.json 2>&1; echo plain rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r01.csv $B > /dev/null 2>&1; echo launches rc=$?
cap() {  # name regex
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:$2" -s 6 -c 1 -o gpurun_out/prof_$1 $B > gpurun_out/ncu_$1.log 2>&1; echo $1 rc=$?
}
cap spmm_fwdout 'GemmCfgILb1ELb0ELb1E.*EpiStoreI13__nv_bfloat16'
cap spmm_pair 'GemmCfgILb1ELb0ELb1E.*EpiStoreIfLb0E'
cap k1 'EpiFwd1'
cap k3 'EpiBwd1'
cap k4 'k_feature_split_x'
