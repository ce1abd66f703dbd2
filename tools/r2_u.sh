set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python tools/graph_vs_eager.py gpt2-xl-dp-d64 3 > gpurun_out/r2u_graph.jsonl 2> gpurun_out/r2u_graph.err
timeout 600 python tools/graph_vs_eager.py bert-large-pp 5 >> gpurun_out/r2u_graph.jsonl 2>> gpurun_out/r2u_graph.err
timeout 600 python tools/graph_vs_eager.py gpt2-xl-dp 3 >> gpurun_out/r2u_graph.jsonl 2>> gpurun_out/r2u_graph.err
timeout 1200 python -m pytest tests/test_parity_gpu.py -q -k "c2" -s > gpurun_out/r2u_c2.log 2>&1
echo "rc=$?" >> gpurun_out/r2u_c2.log
echo done
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:gemm_kernel -s 3 -c 1 \
  -o gpurun_out/r2u_gemm_gelu python tools/gemm_shapes.py ncu 1 > gpurun_out/r2u_ncu_gemm.log 2>&1
echo done2
