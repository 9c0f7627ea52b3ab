cp paper_2306_17486_b200/libhelmsolve_b200.so /tmp/base.so
for v in base na3 base na3; do
  if [ $v = base ]; then cp /tmp/base.so paper_2306_17486_b200/libhelmsolve_b200.so; else cp tools/lib_$v.so paper_2306_17486_b200/libhelmsolve_b200.so; fi
  python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), d['breakdown']['convs']['ms'], d['breakdown']['convs_l0_16ch']['ms'])"
done
cp /tmp/base.so paper_2306_17486_b200/libhelmsolve_b200.so
