timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562 tools/ipc_shard_check.py 20000 10 5 2>&1 | grep "ipc shard check"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29563 tools/ipc_shard_check.py 7001 8 4 2>&1 | grep "ipc shard check"
