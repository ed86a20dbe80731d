# build libfb.so (and optional variants: NAME=-DFLAG ...); non-zero exit on any compile error
cd "$(dirname "$0")/.." || exit 1
python -m paper_2004_09883_b200._build > /tmp/fb_build.log 2>&1 || { grep -iE "error" /tmp/fb_build.log | head; exit 1; }
for v in "$@"; do name=${v%%=*}; flags=${v#*=}; python paper_2004_09883_b200/_build.py --out paper_2004_09883_b200/libfb_$name.so $flags > /tmp/fb_build_$name.log 2>&1 || { grep -iE "error" /tmp/fb_build_$name.log | head; exit 1; }; done
echo build ok
