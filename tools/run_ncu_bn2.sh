# ncu --set full of the fused BN statistics kernel (forward and backward) on the largest SN-GAN layer, 1 GPU
NCU=/usr/local/cuda/bin/ncu
mkdir -p gpurun_out
python tools/bench_bn.py --only 128x128 --dtype f32 --iters 3 > gpurun_out/nbn_plain.txt 2>&1; tail -3 gpurun_out/nbn_plain.txt
timeout 600 $NCU -k regex:bn_stats_fused -c 2 --set full --import-source on --clock-control none -o gpurun_out/ncu_bn_fused python tools/bench_bn.py --only 128x128 --dtype f32 --iters 1 > gpurun_out/ncu_bn_fused.log 2>&1
$NCU -i gpurun_out/ncu_bn_fused.ncu-rep --page raw --csv > gpurun_out/ncu_bn_fused_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/ncu_bn_fused_raw.csv
$NCU -i gpurun_out/ncu_bn_fused.ncu-rep --page details --csv > gpurun_out/ncu_bn_fused_details.csv 2>/dev/null; wc -l gpurun_out/ncu_bn_fused_details.csv
