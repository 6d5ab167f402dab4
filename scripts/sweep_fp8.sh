# Build-time variants of the FP8 engine (ring depth, warps per slot, fold buffers, split P),
# timed on c2 / c3 with an FP8 cache; plus one ncu --set full capture of the default.
mkdir -p /tmp/variants
build() {  # name, defines...
  name=$1; shift
  mkdir -p /tmp/variants/$name
  nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared "$@" -I include \
    paper_2405_10480_b200/csrc/decode.cu paper_2405_10480_b200/csrc/api.cpp paper_2405_10480_b200/csrc/planner.cpp \
    -o /tmp/variants/$name/libleanattn.so 2>/tmp/variants/$name/build.log || echo "build $name failed"
}
run() {  # name, config
  LEANATTN_LIB=/tmp/variants/$1/libleanattn.so timeout 300 python bench.py --config $2 --dtype fp8 --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', '$2', round(r['kernel_us'],1), 'us p10/p50/p90', [round(x,1) for x in r['kernel_us_pct'].values()], round(r['achieved']), 'GB/s', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
build base &
build nosplit -DLA_FP8_SPLITP=0 &
build n5w1 -DLA_FP8_NST=5 -DLA_FP8_WPS=1 &
build n6w1fb1 -DLA_FP8_NST=6 -DLA_FP8_WPS=1 -DLA_FP8_FB=1 &
wait
build n3w3 -DLA_FP8_NST=3 -DLA_FP8_WPS=3 &
build n4w3fb1 -DLA_FP8_NST=4 -DLA_FP8_WPS=3 -DLA_FP8_FB=1 &
build n4w2fb1 -DLA_FP8_NST=4 -DLA_FP8_WPS=2 -DLA_FP8_FB=1 &
build n5w2fb1 -DLA_FP8_NST=5 -DLA_FP8_WPS=2 -DLA_FP8_FB=1 &
wait
grep -h "spill" /tmp/variants/*/build.log | sort | uniq -c | head
for rep in 1 2; do
  for v in base nosplit n5w1 n6w1fb1 n3w3 n4w3fb1 n4w2fb1 n5w2fb1; do run $v c2; run $v c3; done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:la_decode -s 3 -c 1 -o gpurun_out/prof_c2_fp8 python bench.py --dtype fp8 --steps 5 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:la_decode -s 3 -c 1 -o gpurun_out/prof_c3_fp8 python bench.py --config c3 --dtype fp8 --steps 5 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ls gpurun_out
