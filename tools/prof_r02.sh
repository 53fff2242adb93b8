# ncu evidence for profiles/r02: launch list of the bench command (model graph only) + full
# captures of the four ViT-B/16 b256 GEMM shapes (unprotected then protected launch of K1).
mkdir -p gpurun_out/prof2
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/prof2/ncu_launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-campaign > gpurun_out/prof2/bench_under_ncu.log 2>&1
for s in "50432 2304 768 qkv" "50432 768 768 proj" "50432 3072 768 fc1" "50432 768 3072 fc2"; do
  set -- $s
  ncu --set full --clock-control none --import-source on -k regex:gg_protected -s 2 -c 2 \
      -o gpurun_out/prof2/full_$4 python tools/prof_one.py $1 $2 $3 bf16 > /dev/null 2>&1
done
ls -la gpurun_out/prof2
