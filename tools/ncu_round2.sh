# ncu captures for round 2 (one GPU; run each only after the plain command exited 0)
#   bash tools/ncu_round2.sh [tag]
tag=${1:-s2}
mkdir -p gpurun_out
FP64=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum
python tools/one_partition.py C5 > gpurun_out/one_partition_$tag.log 2>&1 || exit 1
# filter + scan of two full-phase balance rounds
timeout 1200 ncu --set full --metrics $FP64 --import-source on --clock-control none \
  -k regex:"filter_kernel|scan_kernel" --launch-skip 892 --launch-count 4 \
  -o gpurun_out/ncu_assign_$tag -f python tools/one_partition.py C5 > gpurun_out/ncu_assign_$tag.log 2>&1
# the movement fold chain of a full-phase iteration
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"run_mark|run_emit|fold_pipe|fold_combine|RadixSort" --launch-skip 300 --launch-count 12 \
  -o gpurun_out/ncu_fold_$tag -f python tools/one_partition.py C5 > gpurun_out/ncu_fold_$tag.log 2>&1
echo ncu_done
