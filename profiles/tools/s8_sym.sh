# linear-molecule (SYM) instance of the 2CLJQ kernel: A/B against the polar-at-COM instance
# (MARDYN_NO_SYM=1) in the same library, and the rigid parity tests
mkdir -p gpurun_out/s8
python -c "import oracle; oracle.build()" > /dev/null 2>&1
for i in 1 2; do for v in 0 1; do
  if [ $v = 1 ]; then export MARDYN_NO_SYM=1; else unset MARDYN_NO_SYM; fi
  python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('no_sym=$v c2', round(d['roofline']['force_ms'],4), round(d['ms_per_step'],4), round(d['value'],1))"
done; done > gpurun_out/s8/ab.log
unset MARDYN_NO_SYM
timeout 1200 python -m pytest tests -m gpu -q -k "c2 or rigid or golden or 2clj or tiny or guard or longrun" > gpurun_out/s8/pytest.log 2>&1
cat gpurun_out/s8/ab.log; tail -2 gpurun_out/s8/pytest.log
