L="1x1_64-256@56 1x1_256-64@56 1x1_128-512@28 1x1_512-128@28"
echo "== default"; python scripts/conv_layers.py $L
echo "== fprop via GEMM"; FP8B_CONV_1X1_GEMM_FPROP=1 python scripts/conv_layers.py $L
echo "== dgrad via GEMM too"; FP8B_CONV_1X1_GEMM_FPROP=1 FP8B_CONV_1X1_GEMM=1 python scripts/conv_layers.py $L
