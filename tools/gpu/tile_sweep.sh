# update times of the bench workload (C2) over PL-NMF tile sizes
for t in ${TILES:-8 10 12 14 16 18 20 24 28 32}; do
  echo "T=$t $(python tools/time_updates.py 26214 11314 1016095 240 $t 2>&1 | grep -E 'update W|update H|iteration' | tr -s ' ' | tr '\n' ' ')"
done
