NCU=/usr/local/cuda/bin/ncu
M="gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed"
timeout 300 $NCU --devices 0 --kernel-name-base demangled -k "regex:k_body<.int.2, .int.4" -c 1 --clock-control none --metrics $M --csv ./tools/nvls_probe 64 > gpurun_out/ncu_nvls_body.csv 2> gpurun_out/ncu_nvls_body.err
timeout 300 $NCU --devices 0 --kernel-name-base demangled -k "regex:k_body<.int.0" -c 1 --clock-control none --metrics $M --csv ./tools/nvls_probe 64 > gpurun_out/ncu_nvls_ldred.csv 2>> gpurun_out/ncu_nvls_body.err
timeout 300 $NCU --devices 0 --kernel-name-base demangled -k "regex:k_body<.int.1" -c 1 --clock-control none --metrics $M --csv ./tools/nvls_probe 64 > gpurun_out/ncu_nvls_st.csv 2>> gpurun_out/ncu_nvls_body.err
# P2P pull / push copy (128-bit peer loads / stores), GPU0 <-> GPU1
timeout 300 $NCU --devices 0 -k regex:k_copy --launch-skip 6 -c 60 --clock-control none --metrics $M --csv ./tools/nvlink_probe > gpurun_out/ncu_p2p_copy.csv 2> gpurun_out/ncu_p2p_copy.err
