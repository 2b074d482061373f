for i in 1 2 3; do
python profiles/time_gram.py 100000000 40,48
KCG_GRAM_HYBRID=1 python profiles/time_gram.py 100000000 40
done
