# fused tensor-core fold raw/plane ring depths on C2 and C4 (diagnostics)
python tools/fold_time.py c2 c4 | sed 's/^/default /'
for d in "8ca172fcfc:-DTC_NR_SELF=3" "95997f944a:-DTC_NR_SELF=4" "46c6c31041:-DTC_NR_SELF=4 -DTC_NP_SELF=3"; do
  tag=${d%%:*}; flags=${d#*:}
  CYC_LIB=paper_2405_16911_b200/_diag/$tag/libcycb200.so CYC_NVCC_EXTRA="$flags" python tools/fold_time.py c2 c4
done
