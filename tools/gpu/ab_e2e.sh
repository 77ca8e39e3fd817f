# A/B of the e2e iterate() loop: HEAD (_ab/) vs the working tree
for i in 1 2; do
echo "HEAD $(cd _ab && python tools/e2e_time.py 2>&1 | tail -1)"
echo "WT   $(python tools/e2e_time.py 2>&1 | tail -1)"
done
