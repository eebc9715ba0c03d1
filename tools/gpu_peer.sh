timeout 900 python -m pytest tests/test_gpu_distributed.py -q -x 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tools/peer_ipc_check.py 2>&1 | grep -v "^\*\|OMP" | tail -5
FMMB_DIST_EXCHANGE=peer timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29632 tools/dist_phases.py c2 5 2>&1 | grep '^{'
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29633 tools/dist_phases.py c2 5 2>&1 | grep '^{'
