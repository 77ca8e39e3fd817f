# A/B of the C5 one-GPU iteration phases: HEAD (built in _ab/) vs the working tree
echo "HEAD"; (cd _ab && timeout 600 python tools/c5_phases.py 2>&1 | tail -4)
echo "WT";   timeout 600 python tools/c5_phases.py 2>&1 | tail -4
