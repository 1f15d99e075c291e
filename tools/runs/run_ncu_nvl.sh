# ncu evidence for the NVLink / NVLS data movement and the fused apply kernel (single-process commands only)
set -x
NCU=/usr/local/cuda/bin/ncu
M="gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed"
# NVLS all-reduce body (ld_reduce + multimem.st), the configuration ar_nvls uses: 148 x 128 threads x 4 in flight
timeout 300 $NCU --devices 0 --kernel-name-base demangled -k "regex:k_body<.int.2, .int.4" -c 1 --clock-control none --metrics $M --csv ./tools/nvls_probe 64 > gpurun_out/ncu_nvls_body.csv 2> gpurun_out/ncu_nvls_body.err
timeout 300 $NCU --devices 0 --kernel-name-base demangled -k "regex:k_body<.int.0" -c 1 --clock-control none --metrics $M --csv ./tools/nvls_probe 64 > gpurun_out/ncu_nvls_ldred.csv 2>> gpurun_out/ncu_nvls_body.err
timeout 300 $NCU --devices 0 --kernel-name-base demangled -k "regex:k_body<.int.1" -c 1 --clock-control none --metrics $M --csv ./tools/nvls_probe 64 > gpurun_out/ncu_nvls_st.csv 2>> gpurun_out/ncu_nvls_body.err
# P2P pull / push copy (128-bit peer loads / stores), GPU0 <-> GPU1
timeout 300 $NCU --devices 0 -k regex:k_copy --launch-skip 6 -c 60 --clock-control none --metrics $M --csv ./tools/nvlink_probe > gpurun_out/ncu_p2p_copy.csv 2> gpurun_out/ncu_p2p_copy.err
# fused apply, 8 virtual replicas, 16M params Adam (HBM-bound form)
timeout 300 python tools/apply_bench.py > gpurun_out/apply_bench_n1.json 2>&1; cat gpurun_out/apply_bench_n1.json
timeout 600 $NCU -k regex:ar_apply -c 1 --set full --import-source on --clock-control none -o /tmp/ncu_apply python tools/apply_bench.py --only fused --steps 1 > gpurun_out/ncu_apply.log 2>&1
$NCU -i /tmp/ncu_apply.ncu-rep --page raw --csv > gpurun_out/ncu_apply_raw.csv 2>/dev/null
$NCU -i /tmp/ncu_apply.ncu-rep --page details --csv > gpurun_out/ncu_apply_details.csv 2>/dev/null
for n in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29514 tools/apply_bench.py > gpurun_out/apply_bench_n$n.json 2> gpurun_out/apply_bench_n$n.err; tail -1 gpurun_out/apply_bench_n$n.json
done
