#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
# the W > 1 code path of the pipelined bench (two ranks on one GPU over CUDA IPC: a code
# path check only -- never a timing)
LG_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/w2_onedev.log 2>&1
echo "w2 exit $?" >> gpurun_out/w2_onedev.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_all.log
timeout 900 python bench.py > gpurun_out/bench_f.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_f.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_qprofile_q -c 1 -s 6 \
    -o gpurun_out/fused_full2 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_fused2.log 2>&1
echo done
