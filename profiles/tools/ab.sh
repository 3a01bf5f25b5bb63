# A/B timing of library variants: LIBS="libmardyn.so libmardyn_b0.so ..." CFGS="c1 c2" bash profiles/tools/ab.sh
LIBS=${LIBS:-"libmardyn.so libmardyn_b0.so"}
for i in 1 2; do for L in $LIBS; do for c in $CFGS; do MARDYN_LIB=$PWD/paper_1408_4599_b200/$L python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(\"$L $c\", round(d[\"roofline\"][\"force_ms\"],4), round(d[\"ms_per_step\"],4))"; done; done; done
