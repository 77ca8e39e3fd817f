# A/B of PLNMF_DBG settings on the W update (tools/time_updates.py)
for d in ${DBGS:-0}; do
  echo "DBG=$d $(PLNMF_DBG=$d python tools/time_updates.py 2>&1 | grep 'update W')"
done
