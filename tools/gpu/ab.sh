# A/B: the committed HEAD (built in _ab/) against the working tree, same box
for i in 1 2 3; do
echo "HEAD    $(cd _ab && python tools/time_updates.py 2>&1 | grep -E "update W|update H" | tr -s " " | tr "\n" " ")"
echo "WT      $(python tools/time_updates.py 2>&1 | grep -E "update W|update H" | tr -s " " | tr "\n" " ")"
done
