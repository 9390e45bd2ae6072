# A/B variants/$V vs the in-tree build on the given configs, then the full GPU suite on the variant
V=$1; shift
bash tools/gpu_ab.sh "$@"
cp paper_2501_17168_b200/libevogp.so /tmp/libevogp.base2.so
cp variants/$V/libevogp.so paper_2501_17168_b200/libevogp.so
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
cp /tmp/libevogp.base2.so paper_2501_17168_b200/libevogp.so
