for i in 1 2; do timeout 300 python scripts/ffn_lab.py README_FFN_ORDER=0,1 8192 2048 32768 2>&1 | tail -1; done
