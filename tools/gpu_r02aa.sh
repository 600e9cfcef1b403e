for rep in 1 2; do
for n in 256 128; do echo "cg n=$n $(timeout 300 python tools/cg_micro.py $n 400 | cut -c1-150)"; done
echo "bi 256 $(timeout 300 python tools/bi_micro.py 256 60 | cut -c100-330)"
echo "bi 128 $(timeout 300 python tools/bi_micro.py 128 60 | cut -c100-330)"
done
