# A/B: HEAD (built in _ab/) vs the working tree on the same box: every kernel family, 3 rounds
for i in 1 2 3; do
echo "HEAD $(cd _ab && python tools/time_updates.py 2>&1 | tr -s ' ' | tr '\n' '|')"
echo "WT   $(python tools/time_updates.py 2>&1 | tr -s ' ' | tr '\n' '|')"
done
