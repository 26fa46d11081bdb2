cd $GRAFT_REPO_ROOT
FP8B_GEMM_EPI=16 timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x -k "lean" 2>&1 | tail -1
for shp in "1048576 512 2048" "1048576 512 1536" "1048576 2048 512" "65536 8192 1024"; do
 set -- $shp
 echo "M=$1 N=$2 K=$3"
 AB_M=$1 AB_NN=$2 AB_K=$3 AB_ROUNDS=4 AB_REPS=5 AB_SLEEP=0.5 timeout 300 python scripts/gemm_ab.py ew8=q:1,FP8B_GEMM_EPI:8,FP8B_GEMM_AST:0 ew16=q:1,FP8B_GEMM_EPI:16,FP8B_GEMM_AST:0 2>&1 | tail -3 | cut -c1-70
done
