set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python bench.py --workload gpt-15b-dp --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/big_15b.json 2> gpurun_out/big_15b.err
timeout 1200 python bench.py --workload resnet-1026-dp --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/big_r1026.json 2> gpurun_out/big_r1026.err
echo done
