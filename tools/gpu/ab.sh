# A/B: the committed HEAD (built in _ab/) against the working tree, same box
echo "HEAD    $(cd _ab && python tools/time_updates.py 2>&1 | grep 'update W')"
echo "WT      $(python tools/time_updates.py 2>&1 | grep 'update W')"
echo HEAD; (cd _ab && PLNMF_PROFILE=1 python tools/profile_step.py 1 2>&1 | grep "W update")
echo WT; PLNMF_PROFILE=1 python tools/profile_step.py 1 2>&1 | grep "W update"
echo HEAD; (cd _ab && PLNMF_TRACE_EXCHANGE=1 python tools/profile_step.py 1 2>&1 | grep -i "exchange\|skew" | head -5)
echo WT; PLNMF_TRACE_EXCHANGE=1 python tools/profile_step.py 1 2>&1 | grep -i "exchange\|skew" | head -5
