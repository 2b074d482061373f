# A/B of the grouped wide Gram's run length (KCG_GROUP_BLOCKS accumulator blocks per warp)
for b in 24 30 36 42; do
  echo "KCG_GROUP_BLOCKS=$b $(KCG_GROUP_BLOCKS=$b python profiles/time_gram.py 20000000 80,96,111,149,160)"
done
