for i in 1 2; do timeout 300 python tools/bench_bn.py --dtype bf16 2>&1 | grep "stats_" | grep -v "H=   8\|H=  16"; echo; done
