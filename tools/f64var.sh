for v in main a b c d; do
  if [ $v = main ]; then L=paper_1607_06283_b200/libevr.so; else L=build_variants/$v.so; fi
  for c in C3 C4 C5; do
    EVR_LIBRARY=$L timeout 300 python bench.py --config $c --precision f64 --no-cpu-baseline --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $c f64', d['ms_per_step'], d['roofline']['frac'])"
  done
done
