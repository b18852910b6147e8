# build the committed HEAD into ab/old (for A/B runs against the working tree)
set -e
rm -rf /tmp/oldrepo; git -C /root/repo worktree prune; git -C /root/repo worktree add -f /tmp/oldrepo HEAD >/dev/null 2>&1
(cd /tmp/oldrepo && python -m paper_2104_13248_b200.build --force >/dev/null)
rm -rf /root/repo/ab/old; mkdir -p /root/repo/ab/old
cp -r /tmp/oldrepo/paper_2104_13248_b200 /tmp/oldrepo/tools /root/repo/ab/old/
echo "ab/old = $(git -C /root/repo rev-parse --short HEAD)"
