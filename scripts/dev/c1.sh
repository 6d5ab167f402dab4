V=paper_2405_10480_b200/lib/variants
for L in $V/r01.so paper_2405_10480_b200/lib/libleanattn.so; do echo "== $L"; LEANATTN_LIB=$L timeout 120 python scripts/tail_report.py c1 2>&1 | head -8; done
