cd /root/repo
for v in head nol1b6 head nol1b6; do AB_ARGS="--steps 10 --warmup 3 --no-frame" tools/ab.sh $v | cut -c1-60; done
AB_ARGS="--steps 30 --warmup 3 --no-frame" tools/ab.sh head nol1b6 | cut -c1-60
