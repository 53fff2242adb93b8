# Final round-2 ncu evidence (profiles/r02/final/): the bench's launch list and full captures of
# the ViT-B/16 b256 GEMM shapes (unprotected then protected K1 launch), fc1 with the fused GELU,
# the tiny (M = 197) int8 launch, and the layer norm.
set -x
D=gpurun_out/prof_final; mkdir -p $D
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $D/ncu_launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-campaign > $D/bench_under_ncu.log 2>&1
for s in "50432 2304 768 bf16 qkv" "50432 768 768 bf16 proj" "50432 3072 768 bf16 fc1" "50432 768 3072 bf16 fc2" \
         "197 768 768 i8 tiny_int8"; do
  set -- $s
  ncu --set full --clock-control none --import-source on -k regex:gg_protected -s 2 -c 2 \
      -o $D/full_$5 python tools/prof_one.py $1 $2 $3 $4 > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:gg_protected -s 2 -c 2 -o $D/full_fc1_gelu \
    python tools/prof_one.py 50432 3072 768 bf16 gelu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:add_layernorm -s 3 -c 1 -o $D/full_ln python tools/prof_ln.py > /dev/null 2>&1
for f in $D/full_*.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}.txt 2>&1; done
rm -f $D/full_qkv.ncu-rep $D/full_fc1.ncu-rep $D/full_fc2.ncu-rep  # summaries kept (64 MiB pull limit)
ls -la $D
