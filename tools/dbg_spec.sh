TTR_QR_TRACE=1 TTR_QR_SPEC_TRACE=1 timeout 900 python - <<'PY' 2>&1 | grep -E "BREAKDOWN|qr speculation" | head -20
import sys; sys.path.insert(0,'.')
import bench, paper_2511_03598_b200 as P
ctx = P.Context(0)
cfg = dict(bench.CFG5B)
x = bench.build_input(P, ctx, cfg)
y = P.round_fixed_krp(x, [cfg["ell"]]*(cfg["d"]-1), 7, rng=P.RNG_PHILOX)
print("done", y.ranks()[:4])
PY
