# bf16 ring-depth variants (GQA c3, MHA c2) after the FP8 findings (deeper ring pays when the
# consumers hold slots longer).
mkdir -p /tmp/variants
build() {
  name=$1; shift
  mkdir -p /tmp/variants/$name
  nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared -Xptxas -v "$@" -I include \
    paper_2405_10480_b200/csrc/decode.cu paper_2405_10480_b200/csrc/api.cpp paper_2405_10480_b200/csrc/planner.cpp \
    -o /tmp/variants/$name/libleanattn.so 2>/tmp/variants/$name/build.log || echo "build $name failed"
}
run() {
  LEANATTN_LIB=/tmp/variants/$1/libleanattn.so timeout 300 python bench.py --config $2 --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', '$2', round(r['kernel_us'],1), 'us p10/p50/p90', [round(x,1) for x in r['kernel_us_pct'].values()], round(r['achieved']), 'GB/s', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
build base &
build g5fb1 -DLA_GQA_NST=5 -DLA_GQA_FB=1 &
build g6w1fb1 -DLA_GQA_NST=6 -DLA_GQA_WPS=1 -DLA_GQA_FB=1 &
build g5w1fb2 -DLA_GQA_NST=5 -DLA_GQA_WPS=1 -DLA_GQA_FB=2 &
wait
build m6w2 -DLA_MHA_NST=6 -DLA_MHA_WPS=2 &
build m6w1 -DLA_MHA_NST=6 -DLA_MHA_WPS=1 &
wait
grep -h "spill" /tmp/variants/m6w2/build.log | sort | uniq -c
for rep in 1 2; do
  for v in base g5fb1 g6w1fb1 g5w1fb2; do run $v c3; done
  for v in base m6w2 m6w1; do run $v c2; done
done
