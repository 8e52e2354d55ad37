# e2e (pinned host buffers) with K2s-c allowed for smaller launches (PD_K2SC_MIN = minimum
# X-masks per launch; default = one residency per ZLO phase: 1184 at N=14, 2368 at N=13)
for n in 14 13; do
  for m in default 512 256 default; do
    if [ $m = default ]; then printf "N=$n K2SC_MIN=default "; PD_N=$n python profiles/scripts/e2e_ab.py;
    else printf "N=$n K2SC_MIN=$m "; PD_K2SC_MIN=$m PD_N=$n python profiles/scripts/e2e_ab.py; fi
  done
done
