# bench.py's N > 1 path at full size on one GPU: ranks as processes on cuda:0, the library's
# NCCL transport through the stand-in (tests/nccl_shim.c).  Correctness / sizing check of the
# multi-GPU bench path, NOT a scaling measurement (the ranks share one GPU and the stand-in
# moves the records through host files).
mkdir -p gpurun_out/s5
gcc -O2 -shared -fPIC -std=gnu11 -I /usr/local/cuda/include -o /tmp/libnccl_shim.so tests/nccl_shim.c -ldl
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export MARDYN_BENCH_ONE_DEVICE=1 MARDYN_NCCL_LIB=/tmp/libnccl_shim.so MDSHIM_DIR=/tmp
python bench.py --config c4 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --rebalance-interval 2 > gpurun_out/s5/c4_n1.json 2> gpurun_out/s5/c4_n1.err
for n in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --config c4 --steps 3 --warmup 3 --e2e-steps 1 --rebalance-interval 2 > gpurun_out/s5/c4_n$n.json 2> gpurun_out/s5/c4_n$n.err
  echo "n=$n rc=$?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config c2 --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/s5/c2_n2.json 2> gpurun_out/s5/c2_n2.err
echo "c2 n=2 rc=$?"
python bench.py --config c2 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/s5/c2_n1.json 2> gpurun_out/s5/c2_n1.err
python - <<'PY'
import json
for f in ["c4_n1", "c4_n2", "c4_n4", "c2_n1", "c2_n2"]:
    try:
        d = json.loads([l for l in open(f"gpurun_out/s5/{f}.json") if l.startswith("{")][0])
        print(f, d["n_gpus"], round(d["value"], 1), d["observables"], "e2e", d["e2e"].get("value") if d["e2e"] else None)
    except Exception as e:
        print(f, "FAILED", e)
PY
for f in gpurun_out/s5/*.err; do echo "== $f"; tail -3 $f; done
