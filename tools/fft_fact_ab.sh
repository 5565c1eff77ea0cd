# factored-twiddle FFT (3 CTAs per SM) vs per-pass tables (diagnostics)
run() { tag=$1; shift; env "$@" ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none -k regex:finalize -s 8 -c 4 --csv python tools/fold_time.py c5 2>/dev/null | grep finalize | awk -F'","' -v t="$tag" '{gsub(/"/,"",$NF); s+=$NF; n++} END {print t, s/n}'; env "$@" python tools/fold_time.py c5 | cut -c1-120 | sed "s/^/$tag /"; }
run fact
run tables CYC_LIB=$(ls -d paper_2405_16911_b200/_diag/*/libcycb200.so | head -1) "CYC_NVCC_EXTRA=-DFFT_FACT=0"
