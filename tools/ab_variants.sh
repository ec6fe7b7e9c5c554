# C3 probe for each library variant under paper_1512_06235_b200/variants (args: names)
mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v"
  MSFM_B200_LIB=$PWD/paper_1512_06235_b200/variants/libmsfm_$v.so timeout 300 python tools/probe_matcher.py 320 0 2>&1 | grep "chunk=\|lines"
done
