mkdir -p gpurun_out/r2f
for v in 0 1 2 3; do echo "== variant $v"; NE_UMMA_VARIANT=$v timeout 120 python tools/umma_diag.py 2>&1 | tail -3; done
NE_IPC_DEBUG=1 timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29915 tools/ipc_debug.py 2 > gpurun_out/r2f/ipc_debug4.log 2>&1; echo rc=$?
grep -v "^ \|^\[ipc" gpurun_out/r2f/ipc_debug4.log | tail -12
for r in 0 1 2 3; do grep "^\[ipc rank $r" gpurun_out/r2f/ipc_debug4.log | tail -4; done
