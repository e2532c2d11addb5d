#!/bin/bash
# ncu evidence for the hot path (run under gpurun on ONE GPU; numbers printed
# under ncu are never bench values). Outputs land in gpurun_out/ncu_<tag>*.
#   tools/ncu_capture.sh <tag> [L H H_kv gain P [attention kernel regex]]
# (the sparse default runs attn64_kernel; dense / > 40 % selected runs attn_kernel)
set -u
cd "$(dirname "$0")/.."
TAG=${1:-r01}
L=${2:-131072}; H=${3:-32}; HKV=${4:-8}; GAIN=${5:-9.0}; P=${6:-0.95}; AK=${7:-attn64_kernel}
mkdir -p gpurun_out
# 1. launch list of one bench step (cold-cache, serialised): per-kernel SHARE of the step
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    -k regex:'attn_kernel|attn64|proxy_kernel|compress_kernel|split_kernel|select|mask_check|finalize|f32_to_bf16|mask_expand' \
    --log-file gpurun_out/ncu_${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-dense --no-parity --also-gain > gpurun_out/ncu_${TAG}_bench_under_ncu.log 2>&1
# 2. full sets: attention (dominant), proxy passes 1+2, compress/split/select
ncu --set full --clock-control none --import-source on -k regex:"$AK" -s 1 -c 1 \
    -o gpurun_out/ncu_${TAG}_attn python tools/profile_case.py $L $H $HKV $GAIN $P > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:proxy -s 2 -c 2 \
    -o gpurun_out/ncu_${TAG}_proxy python tools/profile_case.py $L $H $HKV $GAIN $P > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'compress_kernel|split_kernel|select_fused_kernel' -s 4 -c 4 \
    -o gpurun_out/ncu_${TAG}_small python tools/profile_case.py $L $H $HKV $GAIN $P > /dev/null 2>&1
ls -la gpurun_out/ | grep ncu_${TAG}
