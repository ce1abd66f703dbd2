# round-2 workload evidence: c2 BERT-Large, c3 at D=64, c5 at named depth, the >HBM gpt-15b; ncu launch list
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for w in bert-large-pp gpt2-xl-dp-d64 resnet-1026-dp vgg-416-dp resnet-dp; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2m_bench_$w.json 2> gpurun_out/r2m_bench_$w.err
done
timeout 1200 python bench.py --workload gpt-15b-dp --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2m_bench_gpt-15b-dp.json 2> gpurun_out/r2m_bench_gpt-15b-dp.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/r2m_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2m_ncu_bench.log 2>&1
echo done
