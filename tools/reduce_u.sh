run() { tag=$1; shift; for c in c5 c2; do env "$@" ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none -k regex:reduce -s 8 -c 4 --csv python tools/fold_time.py $c 2>/dev/null | grep reduce | awk -F'","' -v t="$tag $c" '{gsub(/"/,"",$NF); s+=$NF; n++} END {print t, s/n}'; done; }
run u8
run u2 CYC_LIB=paper_2405_16911_b200/_diag/d12e6c04c4/libcycb200.so "CYC_NVCC_EXTRA=-DRED_U=2"
run u4 CYC_LIB=paper_2405_16911_b200/_diag/087d88541a/libcycb200.so "CYC_NVCC_EXTRA=-DRED_U=4"
