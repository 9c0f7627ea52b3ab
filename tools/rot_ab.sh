for lib in "" "--lib tools/_variants/libhelmsolve_b200_norot.so"; do
echo "lib: $lib"
timeout 100 python tools/conv_probe.py --B 64 --H 256 --W 512 --cin 32 --cout 32 --side none --softplus 1 $lib | tail -1
timeout 100 python tools/conv_probe.py --B 64 --H 512 --W 1024 --cin 16 --cout 32 --stride 2 --side none --softplus 1 $lib | tail -1
timeout 100 python tools/conv_probe.py --B 64 --H 256 --W 512 --cin 32 --cout 16 --transposed 1 --stride 2 --side none --softplus 1 $lib | tail -1
timeout 100 python tools/conv_probe.py --B 64 --H 128 --W 256 --cin 64 --cout 32 --transposed 1 --stride 2 --side addend --softplus 1 $lib | tail -1
done
