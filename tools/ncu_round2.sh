# ncu captures for round 2 (one GPU; run each only after the plain command exited 0)
#   bash tools/ncu_round2.sh TAG [ROUND] [FOLD]
tag=${1:-s2}; rnd=${2:-550}; fld=${3:-60}
mkdir -p gpurun_out
FP64=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum
export GP_NVTX=1
python tools/round_trace.py C5 $((rnd-2)) $((rnd+2)) > gpurun_out/round_trace_$tag.txt 2>&1 || exit 1
# filter + scan of one full-phase balance round (NVTX range round<rnd>)
timeout 1200 ncu --nvtx --nvtx-include "round$rnd/" --set full --metrics $FP64 --import-source on \
  --clock-control none -o gpurun_out/ncu_round${rnd}_$tag -f python tools/one_partition.py C5 \
  > gpurun_out/ncu_round_$tag.log 2>&1
# the movement fold chain of one full-phase iteration (NVTX range fold<fld>)
timeout 1200 ncu --nvtx --nvtx-include "fold$fld/" --set full --import-source on --clock-control none \
  -o gpurun_out/ncu_fold${fld}_$tag -f python tools/one_partition.py C5 > gpurun_out/ncu_fold_$tag.log 2>&1
# the bootstrap (keys, sort, gathers, warm-up order) and the delivery
timeout 1200 ncu --nvtx --nvtx-include "bootstrap/" --nvtx-include "deliver/" --section SpeedOfLight \
  --section MemoryWorkloadAnalysis --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -o gpurun_out/ncu_boot_$tag -f python tools/one_partition.py C5 > gpurun_out/ncu_boot_$tag.log 2>&1
echo ncu_done
