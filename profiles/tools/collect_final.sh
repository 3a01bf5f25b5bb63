#!/bin/bash
# Final round-2 bench lines of all five configurations with the final binary, plus the GPU
# test suite and smoke().  Everything lands in gpurun_out/final/.
O=gpurun_out/final; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
python bench.py > $O/bench_c1.json 2> $O/bench_c1.err
for c in c0 c2 c3 c4; do python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
tail -1 $O/smoke.log; tail -1 $O/pytest_gpu.log
