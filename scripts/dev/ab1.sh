V=paper_2405_10480_b200/lib/variants
for c in "--config c1" "--config c2" "--config c3" "--config c4"; do bash scripts/ab_bench.sh "$c" $V/r01.so $V/upd.so cur; done
bash scripts/ab_bench.sh "--config c2 --schedule dynamic --dyn-first 940 --dyn-min 8" cur
