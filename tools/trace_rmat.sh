# per-step timeline of the bench pool's first R-MAT 24 source at the current defaults
DS_DEBUG_PREP=1 python tools/trace_steps.py 2>&1 | grep -v "^\[ds\] launch"
