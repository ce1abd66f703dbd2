set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 120 python tools/gemm_epi_ab.py 4096 1600 1600 >> gpurun_out/r2bb.jsonl 2>>gpurun_out/r2bb.err
HM_GEMM_BN=256 HM_GEMM_CG=2 timeout 120 python tools/gemm_epi_ab.py 4096 1600 1600 >> gpurun_out/r2bb.jsonl 2>>gpurun_out/r2bb.err
HM_GEMM_BN=128 HM_GEMM_CG=2 timeout 120 python tools/gemm_epi_ab.py 4096 1600 1600 >> gpurun_out/r2bb.jsonl 2>>gpurun_out/r2bb.err
HM_GEMM_BN=192 HM_GEMM_CG=1 timeout 120 python tools/gemm_epi_ab.py 4096 1600 1600 >> gpurun_out/r2bb.jsonl 2>>gpurun_out/r2bb.err
timeout 120 python tools/gemm_epi_ab.py 4096 6400 1600 >> gpurun_out/r2bb.jsonl 2>>gpurun_out/r2bb.err
timeout 120 python tools/gemm_epi_ab.py 8192 8192 8192 >> gpurun_out/r2bb.jsonl 2>>gpurun_out/r2bb.err
echo done
