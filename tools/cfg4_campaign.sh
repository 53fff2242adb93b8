# BASELINE configs[3]: ViT-L/16 layer-vulnerability campaigns (fp16: 1e6 trials; tf32: 1e5), one GPU here;
# under torchrun the same entry shards the (layer, block) units and all-reduces the counters (K5).
mkdir -p gpurun_out/cfg4
python -m paper_2310_03841_b200.campaign_vit --model vit_l16 --dtype fp16 --trials 1000000 > gpurun_out/cfg4/vitl_fp16_1e6.json 2> gpurun_out/cfg4/vitl_fp16.err
python -m paper_2310_03841_b200.campaign_vit --model vit_l16 --dtype tf32 --trials 100000 > gpurun_out/cfg4/vitl_tf32_1e5.json 2> gpurun_out/cfg4/vitl_tf32.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    -m paper_2310_03841_b200.campaign_vit --model vit_b16 --dtype bf16 --trials 25600 > gpurun_out/cfg4/vitb_2rank_1gpu.json 2> gpurun_out/cfg4/vitb_2rank.err || true
