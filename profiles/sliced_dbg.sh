for a in "40 129" "40 300" "40 20000" "40 200000" "40 2000000" "17 2000000" "24 2000000"; do KCG_GRAM_SLICED=1 timeout 60 python profiles/sliced_dbg.py $a 2>&1 | tail -2; done
