set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/cublas_shapes.py > gpurun_out/r2t_cublas.jsonl 2> gpurun_out/r2t_cublas.err
timeout 300 python tools/gemm_shapes.py ours > gpurun_out/r2t_ours.jsonl 2>> gpurun_out/r2t_cublas.err
echo done
