for lib in libtsds libtsds_mb3 libtsds_noL1 libtsds_mb3noL1; do
  echo "== $lib"
  export TSDS_LIB=$PWD/paper_2307_05389_b200/$lib.so
  python tools/variants.py c2 20 2>&1 | grep ldg
  python tools/variants.py c1 50 2>&1 | grep ldg
  C5_S=1024 python tools/variants.py c5i16 10 2>&1 | grep ldg
  C5_S=1024 python tools/variants.py c5u8 10 2>&1 | grep ldg
done
