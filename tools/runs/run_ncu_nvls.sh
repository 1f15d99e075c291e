NCU=/usr/local/cuda/bin/ncu
M="gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for sel in "k_body<.int.2, .int.4" "k_body<.int.0" "k_body<.int.1"; do
timeout 600 $NCU --replay-mode application --devices 0 --kernel-name-base demangled -k "regex:$sel" -c 1 --clock-control none --metrics $M --csv ./tools/nvls_probe 64 2>&1 | grep -v "^ldred\|^ld_reduce\|^st \|^kernel\|GPUs," | tail -12
done
