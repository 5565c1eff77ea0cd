# split_planes samples per thread (diagnostics): kernel time (ncu, warm) and the C5 step
run() { tag=$1; shift; env "$@" ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none -k regex:split -s 4 -c 3 --csv python tools/fold_time.py c5 2>/dev/null | grep split | awk -F'","' -v t="$tag" '{gsub(/"/,"",$NF); s+=$NF; n++} END {print t, s/n}'; }
run s4
run s1 CYC_LIB=paper_2405_16911_b200/_diag/fd12d0c992/libcycb200.so "CYC_NVCC_EXTRA=-DSPLIT_S=1"
run s2 CYC_LIB=paper_2405_16911_b200/_diag/ca04c3630e/libcycb200.so "CYC_NVCC_EXTRA=-DSPLIT_S=2"
run s8 CYC_LIB=paper_2405_16911_b200/_diag/02216e4819/libcycb200.so "CYC_NVCC_EXTRA=-DSPLIT_S=8"
