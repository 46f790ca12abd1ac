# Round-2e: config-5 certificate (reduced n first as a script check, then full size)
set -x
true

timeout 4000 python tests/tools/cfg5_certificate.py --out gpurun_out/cfg5_certificate.json > gpurun_out/cert_full.log 2>&1; echo full_rc=$?
tail -3 gpurun_out/cert_full.log
free -g
