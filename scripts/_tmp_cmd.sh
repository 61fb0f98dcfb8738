bash scripts/ab_run.sh ab13 cur curnost curmem
bash scripts/probe_timing.sh ab13 curtim
