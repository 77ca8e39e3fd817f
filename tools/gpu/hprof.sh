# Developer build (_dbg/, -DPLNMF_DEBUG_KNOBS): per-section cycle profile of the H and W updates at C2,
# and the update times with the look-ahead skipped / not overlapped
cd _dbg
PLNMF_PROFILE=1 python tools/profile_step.py 3 2>&1 | tail -8
for kn in "" PLNMF_SKIP_LOOKAHEAD PLNMF_NO_OVERLAP; do
  echo "knob=$kn $(env $kn${kn:+=1} python tools/time_updates.py 2>&1 | grep -E 'update W|update H' | tr -s ' ' | tr '\n' ' ')"
done
