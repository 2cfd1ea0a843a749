python paper_2411_15997_b200/build.py >/dev/null
for j in 2 4 8 16 64 256; do echo "JACOBI_MAX=$j"; FS_ACT_JACOBI_MAX=$j python tools/prof_stages.py c3 2>&1 | grep -E "act |act_walk|act_decide"; done
