mkdir -p gpurun_out/prof3
python tools/prof_ln.py > gpurun_out/prof3/ln_time.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:add_layernorm -s 3 -c 1 -o gpurun_out/prof3/full_ln python tools/prof_ln.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gg_protected -s 2 -c 2 -o gpurun_out/prof3/full_fc1_gelu python tools/prof_one.py 50432 3072 768 bf16 gelu > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gg_protected --csv python tools/prof_one.py 50432 3072 768 bf16 gelu > gpurun_out/prof3/fc1_gelu_times.csv 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gg_protected --csv python tools/prof_one.py 50432 3072 768 bf16 > gpurun_out/prof3/fc1_times.csv 2>&1
python -m paper_2310_03841_b200.campaign_vit --model vit_l16 --dtype fp16 --trials 20000 > gpurun_out/prof3/campaign_l16_small.json 2> gpurun_out/prof3/campaign_l16_small.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-campaign > gpurun_out/prof3/bench.json 2> gpurun_out/prof3/bench.err
