# split beside the fold (timing probe; DIAG_SPLIT_ASYNC results are wrong) and split grid sizes
run() { tag=$1; shift; env "$@" python tools/fold_time.py c5 | sed "s/^/$tag /" | cut -c1-170; }
run default
run grid296 CYC_LIB=paper_2405_16911_b200/_diag/7837fb8950/libcycb200.so "CYC_NVCC_EXTRA=-DSPLIT_GRID=296"
run async148 CYC_LIB=paper_2405_16911_b200/_diag/f420434cd6/libcycb200.so "CYC_NVCC_EXTRA=-DDIAG_SPLIT_ASYNC -DSPLIT_GRID=148"
run async296 CYC_LIB=paper_2405_16911_b200/_diag/657eeebae3/libcycb200.so "CYC_NVCC_EXTRA=-DDIAG_SPLIT_ASYNC -DSPLIT_GRID=296"
run asyncall CYC_LIB=paper_2405_16911_b200/_diag/61f2e59c8d/libcycb200.so "CYC_NVCC_EXTRA=-DDIAG_SPLIT_ASYNC -DSPLIT_GRID=65536"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:split -s 4 -c 2 --csv python tools/fold_time.py c5 2>/dev/null | grep split | awk -F'","' '{gsub(/"/,"",$NF); print "split(default grid) ns", $NF}'
