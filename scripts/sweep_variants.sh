# Build-time ring / warp variants of the decode kernel, timed on c2 (MHA) and c3 (GQA).

mkdir -p /tmp/variants
build() {  # name, defines...
  name=$1; shift
  mkdir -p /tmp/variants/$name
  nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared "$@" -I include \
    paper_2405_10480_b200/csrc/decode.cu paper_2405_10480_b200/csrc/api.cpp paper_2405_10480_b200/csrc/planner.cpp \
    -o /tmp/variants/$name/libleanattn.so
}
run() {  # name, config
  LEANATTN_LIB=/tmp/variants/$1/libleanattn.so timeout 300 python bench.py --config $2 --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', '$2', round(d['roofline']['kernel_us'],1), 'us', round(d['roofline']['achieved']), 'GB/s', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
}
build base
build g4fb2 -DLA_GQA_NST=4 -DLA_GQA_FB=2
build g6w1 -DLA_GQA_NST=6 -DLA_GQA_WPS=1 -DLA_GQA_FB=1
build gnosplit -DLA_GQA_SPLITP=0
build m6w1 -DLA_MHA_NST=6 -DLA_MHA_WPS=1
build m4w2 -DLA_MHA_NST=4 -DLA_MHA_WPS=2
for v in base g4fb2 g6w1 gnosplit; do run $v c3; done
for v in base m6w1 m4w2; do run $v c2; done
for v in base g4fb2 g6w1 gnosplit; do run $v c3; done
for v in base m6w1 m4w2; do run $v c2; done
