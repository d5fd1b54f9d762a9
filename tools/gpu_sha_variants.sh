for v in default s4c2 s5c2 s6c2; do
  L=""; [ $v != default ] && L=$PWD/tools/micro/libpolar_$v.so
  echo "== $v B=64 Hkv=32"; PS_LIB_PATH=$L SHORT=1 SPLITS=0,-296,-592,-888 python tools/sha_k.py
  echo "== $v B=128 Hkv=32"; PS_LIB_PATH=$L SHORT=1 B=128 SPLITS=0,-296,-592 python tools/sha_k.py
  echo "== $v B=64 Hkv=8"; PS_LIB_PATH=$L SHORT=1 H_KV=8 SPLITS=0,-296,-592 python tools/sha_k.py
  echo "== $v B=256 Hkv=8"; PS_LIB_PATH=$L SHORT=1 B=256 H_KV=8 SPLITS=0,-296,-592 python tools/sha_k.py
done
