# ncu evidence for profiles/: launch list of the bench command + full captures of the four
# ViT-B/16 b256 GEMM shapes (unprotected then protected launch of the same kernel family).
set -e
mkdir -p gpurun_out/prof
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gg_protected -c 800 --csv --log-file gpurun_out/prof/ncu_launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_under_ncu.log 2>&1
for s in "50432 2304 768 qkv" "50432 768 768 proj" "50432 3072 768 fc1" "50432 768 3072 fc2"; do
  set -- $s
  ncu --set full --clock-control none --import-source on -k regex:gg_protected -s 2 -c 2 \
      -o gpurun_out/prof/full_$4 python tools/prof_one.py $1 $2 $3 bf16 > /dev/null 2>&1
done
