# FP8 engine, second sweep: MHA (1-row fold) ring depth, GQA default vs split P.
mkdir -p /tmp/variants
build() {
  name=$1; shift
  mkdir -p /tmp/variants/$name
  nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared "$@" -I include \
    paper_2405_10480_b200/csrc/decode.cu paper_2405_10480_b200/csrc/api.cpp paper_2405_10480_b200/csrc/planner.cpp \
    -o /tmp/variants/$name/libleanattn.so 2>/tmp/variants/$name/build.log || echo "build $name failed"
}
run() {
  LEANATTN_LIB=/tmp/variants/$1/libleanattn.so timeout 300 python bench.py --config $2 --dtype fp8 --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', '$2', round(r['kernel_us'],1), 'us p10/p50/p90', [round(x,1) for x in r['kernel_us_pct'].values()], round(r['achieved']), 'GB/s', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fp8.py -q -x 2>&1 | tail -3
build base &
build m5fb2 -DLA_FP8M_NST=5 &
build m6fb1 -DLA_FP8M_FB=1 &
build m4w3 -DLA_FP8M_NST=4 -DLA_FP8M_WPS=3 &
build gsplit -DLA_FP8_SPLITP=1 &
build g4fb2 -DLA_FP8_NST=4 -DLA_FP8_FB=2 &
wait
for rep in 1 2; do
  for v in base m5fb2 m6fb1 m4w3 gsplit; do run $v c2; done
  for v in base gsplit g4fb2; do run $v c3; done
done
