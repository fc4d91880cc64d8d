g++ -std=c++17 -O2 -fPIC -shared -o /tmp/libfakenccl.so tests/fake_nccl/fake_nccl.cpp -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart -lrt
export B2M_NCCL_LIB=/tmp/libfakenccl.so
for t in 1 2 3 4 5 6; do
rm -rf /tmp/w3; mkdir -p /tmp/w3
for r in 0 1 2; do timeout 40 python tests/nccl_world_worker.py $r 3 2958$t /tmp/w3 3 ok > /tmp/w3/log$r 2>&1 & done
wait
n=$(ls /tmp/w3/*.npz 2>/dev/null | wc -l)
echo "=== trial $t: $n npz"
if [ "$n" != "3" ]; then cat /tmp/w3/*.err 2>/dev/null; for r in 0 1 2; do echo "== rank $r"; grep -v "^\s*$\|allreduce\|init done" /tmp/w3/log$r | tail -24; done; break; fi
done
