for c in 1 2 4 8; do
  echo "C=$c" >> gpurun_out/rowc.txt
  FQ_ROW_C=$c python scripts/hars_ab.py 2>&1 | cut -c1-400 >> gpurun_out/rowc.txt
done
