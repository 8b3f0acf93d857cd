# parity tests under several kernel configurations (env TESTCFG="A=1 B=2;C=3")
IFS=';' read -ra VS <<< "${TESTCFG:-SGM_BULK=1}"
for V in "${VS[@]}"; do
  echo "== $V"
  env $V python -m pytest tests -m gpu -q -x ${PYARGS} 2>&1 | tail -4
done
