for d in 4 5 20 13 15; do echo "dbg=$d"; CIRR_QR_DBG=$d timeout 120 python -c "
import sys; sys.path.insert(0,'tools'); import qr_ab
for k in (120,256):
    l,i,t,q,A,B=qr_ab.run(k,2,False,0)
    r=q[1]
    print(k, '%.2f ms'%t, 'sweeps',q[0],'rot',r,'chain cyc/rot %.0f'%(q[3]/r), 'wait %.0f issue %.0f front %.0f rest %.0f'%((q[5]&0xffffffff)/r,(q[5]>>32)/r,q[6]/r,q[7]/r))
"; done
