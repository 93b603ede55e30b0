#!/usr/bin/env bash
# Round-end checks in ONE gpurun call, run HERE (reads /root/reference for the
# reference's own test files, which travel inside the command; see
# run_reference_tests.sh): the reference's tests against the package, every
# BASELINE config shape (tools/configs.sh), and bench.py under a 1-rank
# torchrun (the NCCL communicator, barriers and final all-reduces on a B200).
set -euo pipefail
files="conftest.py test_scan.py test_mesh.py test_normals.py test_segment.py test_simulate.py test_evaluate.py"
blob=$(tar -C /root/reference/pkg/tests -cJf - $files | base64 -w0)
exec /usr/local/graft/bin/gpurun --timeout 1800 -- "mkdir -p gpurun_out /tmp/lidarseg_reftests && \
echo $blob | base64 -d | tar -C /tmp/lidarseg_reftests -xJf - && \
(PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=\$GRAFT_REPO_ROOT/tools/refshim:\$GRAFT_REPO_ROOT \
timeout 1000 python -m pytest -p no:cacheprovider -v -rA /tmp/lidarseg_reftests > gpurun_out/reftests.log 2>&1; \
tail -3 gpurun_out/reftests.log); \
bash tools/configs.sh > gpurun_out/configs.txt 2>&1; cat gpurun_out/configs.txt | cut -c1-150; \
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline --no-latency --no-accuracy \
> gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err; echo torchrun rc=\$?; \
grep -E 'NCCL INFO (comm|ncclCommInit|Init)' gpurun_out/torchrun1.err | head -5; tail -c 300 gpurun_out/torchrun1.json"
