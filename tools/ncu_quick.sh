#!/bin/bash
# usage: tools/ncu_quick.sh TAG KERNEL_REGEX [env...] -- quick ncu counters (time, DRAM bytes, FMA pipe, issue,
# top stalls) of one K1 launch at cfg4; writes gpurun_out/q_TAG.csv
TAG=$1; KRE=$2; shift 2
env "$@" ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sector_op_read_hit_rate.pct,smsp__average_warp_latency_issue_stalled_no_instructions.ratio,launch__registers_per_thread --clock-control none -k regex:$KRE -s 2 -c 1 --csv python tools/profile_k1.py cfg4 4 > gpurun_out/q_$TAG.csv 2>/dev/null
grep -E "gpu__time|dram__bytes|fma_cycles|issue_active|hit_rate|no_instr|registers" gpurun_out/q_$TAG.csv | awk -F'","' -v t=$TAG '{print t, $(NF-2), $NF}'
