# Round-2x: the SURVEY 8(c) config-5 full-size host certificate re-run on HEAD (coefficient kernel, pair post-step,
# selected-vector Rayleigh-Ritz and the 4-stage Ritz ring changed since profiles/r2q_cfg5_certificate.json)
set -x
timeout 2300 python tests/tools/cfg5_certificate.py --out gpurun_out/r2x_cfg5_certificate.json > gpurun_out/r2x_cfg5_certificate.log 2>&1; echo cert_rc=$?
tail -n 2 gpurun_out/r2x_cfg5_certificate.log | cut -c1-600
