# build the working tree with extra nvcc flags into ab/<name>:  tools/ab/ab_variant.sh NAME "-DFOO=1"
set -e
name=$1; extra=$2
d=/tmp/var_$name; rm -rf $d; mkdir -p $d
cp -r /root/repo/paper_2104_13248_b200 /root/repo/tools /root/repo/include $d/
rm -f $d/paper_2104_13248_b200/libconebp_b200.so
(cd $d && CBP_NVCC_EXTRA="$extra" python -m paper_2104_13248_b200.build --force >/dev/null)
rm -rf /root/repo/ab/$name; mkdir -p /root/repo/ab/$name
cp -r $d/paper_2104_13248_b200 $d/tools /root/repo/ab/$name/
echo "ab/$name built with $extra"
