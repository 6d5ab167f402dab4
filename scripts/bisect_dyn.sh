# Build older library versions (variants_src/<commit>, untracked) and time c3/c2 dynamic vs static.
for c in $(ls variants_src); do
  mkdir -p /tmp/variants/$c
  nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared -I variants_src/$c/include \
    variants_src/$c/paper_2405_10480_b200/csrc/decode.cu variants_src/$c/paper_2405_10480_b200/csrc/api.cpp \
    variants_src/$c/paper_2405_10480_b200/csrc/planner.cpp -o /tmp/variants/$c/libleanattn.so &
done
wait
for c in $(ls variants_src); do
  for s in streamk dynamic; do
    LEANATTN_LIB=/tmp/variants/$c/libleanattn.so timeout 300 python bench.py --config c3 --schedule $s --steps 100 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | \
      python -c "import json,sys; t=sys.stdin.read(); d=json.loads(t) if t.startswith('{') else None; print('$c', 'c3', '$s', round(d['roofline']['kernel_us'],1) if d else t[:200])"
  done
done
