for i in 1 2; do
echo "HEAD $(cd _ab && python tools/time_updates.py 2>&1 | grep -E "update W|iteration" | tr -s " " | tr "\n" " ")"
for v in s0 1 2 16; do echo "v$v   $(cd _v$v && python tools/time_updates.py 2>&1 | grep -E "update W|iteration" | tr -s " " | tr "\n" " ")"; done
done
