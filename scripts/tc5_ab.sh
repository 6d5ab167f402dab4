# A/B of two libleanattn builds on one box: c3 N_q=Q, alternating, 3 rounds each
A=${A:-paper_2405_10480_b200/lib/libleanattn.so}; B=${B:-variants/libla_noldefer.so}; Q=${Q:-4}
for r in 1 2 3; do for L in $A $B; do
LEANATTN_LIB=$L timeout 120 python bench.py --config c3 --q-len $Q --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'$L'", d["ms_per_step"])'
done; done
