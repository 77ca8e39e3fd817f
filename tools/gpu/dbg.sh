for d in 0 15; do for s in 0 1; do
  if [ $s = 1 ]; then export PLNMF_SKIP_LOOKAHEAD=1; else unset PLNMF_SKIP_LOOKAHEAD; fi
  echo "DBG=$d SKIP=$s $(PLNMF_DBG=$d python tools/time_updates.py 2>&1 | grep 'update W')"
done; done
