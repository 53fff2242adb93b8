# BASELINE configs[3]: ViT-L/16 layer-vulnerability campaigns, one GPU here; under torchrun the same
# entry shards the (layer, block) units over the ranks and all-reduces the counters (K5).
# Golden set: images the fp16 / tf32 model classifies like its fp32 teacher, top-2 gap > 2 ulps.
mkdir -p gpurun_out/cfg4
python -m paper_2310_03841_b200.campaign_vit --model vit_l16 --dtype fp16 --trials 1000000 > gpurun_out/cfg4/vitl_fp16_1e6.json 2> gpurun_out/cfg4/vitl_fp16.err
python -m paper_2310_03841_b200.campaign_vit --model vit_l16 --dtype fp16 --trials 200000 --modes random_value > gpurun_out/cfg4/vitl_fp16_rv_2e5.json 2> gpurun_out/cfg4/vitl_fp16_rv.err
python -m paper_2310_03841_b200.campaign_vit --model vit_l16 --dtype tf32 --trials 100000 --modes random_value > gpurun_out/cfg4/vitl_tf32_rv_1e5.json 2> gpurun_out/cfg4/vitl_tf32.err
