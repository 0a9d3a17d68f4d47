bash scripts/ab_libs.sh ab_deep5c 5 2
