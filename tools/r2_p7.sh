# the N>1 bench path on one GPU (gloo + host communicator), then the default lines
O=gpurun_out/p7; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611"
timeout 600 $TR bench.py --gpus 2 --steps 5 --warmup 3 --transport host --no-e2e --no-cpu-baseline > $O/n2_weak.json 2> $O/n2_weak.err; echo "weak rc=$?"
timeout 600 $TR bench.py --gpus 2 --steps 5 --warmup 3 --transport host --no-e2e --no-cpu-baseline --config config4 --global-batch 1024 --mode fused > $O/n2_strong4.json 2> $O/n2_strong4.err; echo "strong4 rc=$?"
timeout 600 $TR bench.py --gpus 2 --steps 5 --warmup 3 --transport host --no-e2e --no-cpu-baseline --config config4 --global-batch 1024 --mode fused --combine peer > $O/n2_strong4_peer.json 2> $O/n2_strong4_peer.err; echo "peer rc=$?"
timeout 600 $TR bench.py --gpus 2 --steps 5 --warmup 3 --transport host --no-e2e --no-cpu-baseline --combine peer > $O/n2_weak_peer.json 2> $O/n2_weak_peer.err; echo "weakpeer rc=$?"
timeout 600 $TR bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > $O/n2_ref.json 2> $O/n2_ref.err; echo "ref2 rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/n1.json 2> $O/n1.err; echo "n1 rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref1.json 2> $O/ref1.err; echo "ref1 rc=$?"
