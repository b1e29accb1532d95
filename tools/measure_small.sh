python -m pytest tests -m gpu -x -q -k "chol or orth or cholqr2" 2>&1 | tail -1
echo chol_small b=20,50,64,112:
ncu --metrics gpu__time_duration.sum --csv python tools/chol_bench.py 2>/dev/null | grep chol_small | awk -F'","' '{print $NF}' | tr '\n' ' '; echo
echo panel 1e5x50:; ncu --metrics gpu__time_duration.sum --csv python tools/panel_one.py 100000 50 2 2>/dev/null | grep cholqr2 | awk -F'","' '{print $NF}' | tr '\n' ' '; echo
echo panel 1e5x100:; ncu --metrics gpu__time_duration.sum --csv python tools/panel_one.py 100000 100 2 2>/dev/null | grep cholqr2 | awk -F'","' '{print $NF}' | tr '\n' ' '; echo
echo chol_wide 2000:; ncu --metrics gpu__time_duration.sum --csv python tools/chol_wide_one.py 2000 2 2>/dev/null | grep chol_wide_kernel | awk -F'","' '{print $NF}' | tr '\n' ' '; echo
