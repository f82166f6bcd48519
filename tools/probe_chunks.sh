# C3 init time vs upload chunk size (GSGP_UPLOAD_CHUNK cases; default 48 MB of rows)
for ch in default 1333248 2666496 12500000; do
  if [ "$ch" = default ]; then unset GSGP_UPLOAD_CHUNK; else export GSGP_UPLOAD_CHUNK=$ch; fi
  echo "chunk=$ch $(timeout 300 python tools/probe_interp.py c3 2 2>&1 | tail -1)"
done
