bash tools/ab.sh ab13c4 4 2 base slot32 slot64
bash tools/ab.sh ab13 2 1 base slot32
