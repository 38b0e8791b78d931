# brute-force tile variants: sources per thread x packed lanes (W1G_TILE_RFULL, W1G_TILE_PACKQ)
for r in 8 16; do for p in 0 1; do
  echo "R=$r PACKQ=$p $(W1G_TILE_RFULL=$r W1G_TILE_PACKQ=$p python tools/micro/brute_tile.py 1000000) $(W1G_TILE_RFULL=$r W1G_TILE_PACKQ=$p python tools/micro/brute_tile.py 100000)"
done; done
