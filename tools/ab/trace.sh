for wl in 80 160; do
for env in "HTG_FDM_TEAM=2" "HTG_FDM_TEAM=3 HTG_FDM_NTEAMS=5" "HTG_FDM_TEAM=4"; do
echo "== wl $wl $env"
env $env HTG_LIB=exp/fdmtrace.so python tools/run_once.py --what sweep --reps 3 --wavelengths $wl 2>&1 | grep "fdm trace" | tail -32 | grep "part 0" | sort -k4n -k6n
done; done
