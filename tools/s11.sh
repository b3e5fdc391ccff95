timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -4
tools/ab.sh "base slowtanh" "colreduce ln_gelu bert" 2
