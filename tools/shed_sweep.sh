for c in 15 7 3; do for e in 64 16 4; do
  echo "== check=$c export=$e"; VCG_WCHECK=$c VCG_WEXPORT=$e timeout 100 python tools/tail_probe.py | grep "^k=" | awk '{print $1, $2, $3, $7, $8}' | sed -n '1p;4p;5p'
done; done
