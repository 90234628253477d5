# 4 GPUs: c2 async (LocalSGD, tau=10) and FedAdam, and c4 sync (fused exchange)
tr() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 4 --no-e2e "$@"; }
tr --mode async --tau 10 > gpurun_out/m4_async.json 2> gpurun_out/m4_async.err; echo "async rc=$?"
tr --mode fedadam --tau 10 > gpurun_out/m4_fedadam.json 2> gpurun_out/m4_fedadam.err; echo "fedadam rc=$?"
tr --config c4 --steps 5 > gpurun_out/m4_c4.json 2> gpurun_out/m4_c4.err; echo "c4 rc=$?"
